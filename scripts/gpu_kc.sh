# kc > k colours: parity; regression of the whole quick suite
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "not config3_full" 2>&1 | tail -4
timeout 900 python scripts/agg_sweep.py --config 3 --envs "CC_COMBINE_IMPL=z" 2>&1 | tail -1
