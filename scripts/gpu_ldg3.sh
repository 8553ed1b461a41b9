# lean gather with L2 hints: parity, sweep of row depth x hub fraction
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 1500 python scripts/agg_sweep.py --config 3 --check --envs "CC_LDG_VARIANT=0,2;CC_HUB_L2_FRAC=0,0.3,0.6,0.9" 2>&1 | tail -8
timeout 900 python scripts/agg_sweep.py --config 3 --precision fp64 --envs "CC_LDG_VARIANT=0,1,2;CC_HUB_L2_FRAC=0.6" 2>&1 | tail -3
