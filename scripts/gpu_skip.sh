# sector skipping of entries no destination of that colour can use
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x -k "not full_size and not config3" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --check --reps 3 --envs "CC_SECTOR_SKIP=0,1" 2>&1 | tail -2 | cut -c1-300
timeout 900 python scripts/agg_sweep.py --config 3 --precision fp64 --check --reps 2 --envs "CC_SECTOR_SKIP=0,1" 2>&1 | tail -2 | cut -c1-300
timeout 1500 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c4', d['ms_per_step'], d['phase_ms'])"
timeout 1800 python -m pytest tests/test_gpu_config4.py -m gpu -q -x 2>&1 | tail -2
