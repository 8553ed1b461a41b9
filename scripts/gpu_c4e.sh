# fp32 shared-memory N'' rows for wide rows (config 4 occupancy)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 1500 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4e.log 2>&1; echo c4 rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_c4e.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phase_ms'], d['roofline'])"
timeout 1800 python -m pytest tests/test_gpu_config4.py -m gpu -q -x 2>&1 | tail -2
