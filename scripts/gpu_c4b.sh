# config 4 on one GPU with the current kernels (+ combine variants); ncu of k_csort2 on config 3
mkdir -p gpurun_out
timeout 1500 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4b.log 2>&1; echo c4 rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_c4b.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phase_ms'], d['peak_table_bytes'])"
CC_COMBINE_V=1 timeout 1500 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4c.log 2>&1; echo c4v1 rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_c4c.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phase_ms'])"
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD1 > gpurun_out/plain_cs.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_csort2 -c 1 -o gpurun_out/csort2 $CMD1 > gpurun_out/ncu_cs.log 2>&1; echo full rc=$?
