# combine with 2 vertices per lane; MoM estimator test
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_COMBINE_V=1,2" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 2 --check --envs "CC_COMBINE_V=1,2;CC_COMBINE_IMPL=lane,tile" 2>&1 | tail -4
timeout 900 python scripts/agg_sweep.py --config 1 --precision fp64 --check --envs "CC_COMBINE_V=1,2;CC_COMBINE_IMPL=lane,tile" 2>&1 | tail -4
