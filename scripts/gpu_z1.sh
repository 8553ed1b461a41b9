# Z-block register-blocked combine: parity, combine sweep, config 4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_COMBINE_IMPL=z,lane" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 2 --check --envs "CC_COMBINE_IMPL=z,lane,tile" 2>&1 | tail -3
timeout 900 python scripts/agg_sweep.py --config 2 --precision fp64 --check --envs "CC_COMBINE_IMPL=z,lane,tile" 2>&1 | tail -3
timeout 1500 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4z.log 2>&1; echo c4 rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_c4z.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phase_ms'])"
