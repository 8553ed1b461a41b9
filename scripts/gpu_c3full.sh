# configs[3] at full size vs the oracle (host DP, double)
mkdir -p gpurun_out
free -g | head -2
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k config3_full --durations=3 2>&1 | tail -6
