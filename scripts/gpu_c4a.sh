# 16-warp lane combine; configs[4] at full size on one GPU (sampled-row parity)
mkdir -p gpurun_out
free -g | head -2; nproc; nvidia-smi --query-gpu=memory.total,memory.used --format=csv
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_COMBINE_IMPL=tile,lane" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --precision fp64 --check --envs "CC_COMBINE_IMPL=tile,lane" 2>&1 | tail -2
timeout 1800 python -m pytest tests/test_gpu_config4.py -m gpu -q -x -s 2>&1 | tail -15
timeout 1200 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4 rc=$?; tail -c 1500 gpurun_out/bench_c4.log
