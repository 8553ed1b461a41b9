# csort small-item kernel: parity and timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_CSORT_SMALL=0,1" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 2 --check --envs "CC_CSORT_SMALL=0,1" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 1 --precision fp64 --check --envs "CC_CSORT_SMALL=0,1" 2>&1 | tail -2
