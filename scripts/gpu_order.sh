# internal vertex order: degree-descending (default) vs original ids
mkdir -p gpurun_out
timeout 900 python scripts/agg_sweep.py --config 3 --envs "CC_LDG_VARIANT=0" 2>&1 | tail -1
CC_ORDER=id timeout 900 python scripts/agg_sweep.py --config 3 --envs "CC_LDG_VARIANT=0" 2>&1 | tail -1
timeout 900 python scripts/agg_sweep.py --config 2 --envs "CC_LDG_VARIANT=0" 2>&1 | tail -1
CC_ORDER=id timeout 900 python scripts/agg_sweep.py --config 2 --envs "CC_LDG_VARIANT=0" 2>&1 | tail -1
