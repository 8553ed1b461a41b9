# random-row gather ceiling microbenchmark; csort batching; e2e
mkdir -p gpurun_out
timeout 600 ./scripts/micro/rowgather 2>&1 | tee gpurun_out/rowgather.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_micro.log; cut -c1-300 gpurun_out/bench_micro.log
python -c "import json;d=json.loads(open('gpurun_out/bench_micro.log').read());print(d['phase_ms'], d['e2e'])"
