# lean cp.async ring for wide rows; narrow D=3 variant; e2e with device-side colour permutation
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 1200 python scripts/agg_sweep.py --config 3 --check --envs "CC_LDG_VARIANT=0,10,11" 2>&1 | tail -3
timeout 900 python scripts/agg_sweep.py --config 3 --envs "CC_RING_VARIANT=0,2" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --precision fp64 --check --envs "CC_LDG_VARIANT=0,10,11" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
