# pipelined lane combine: parity, combine sweep vs the V-tile kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_COMBINE_IMPL=tile,lane" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --precision fp64 --check --envs "CC_COMBINE_IMPL=tile,lane" 2>&1 | tail -2
timeout 600 python scripts/agg_sweep.py --config 2 --check --envs "CC_COMBINE_IMPL=tile,lane" 2>&1 | tail -2
timeout 600 python scripts/agg_sweep.py --config 1 --check --envs "CC_COMBINE_IMPL=tile,lane" 2>&1 | tail -2
