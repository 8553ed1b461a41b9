# sibling-pair gather: parity subset, A/B bench, TMA gather4 microbenchmark, launch list
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x -k "sibling or knob or twins or config0 or small_suite or fused" > gpurun_out/pytest_pair.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_pair.log
timeout 300 ./scripts/micro/tma_gather4 > gpurun_out/tma_gather4.log 2>&1; echo micro rc=$?; cat gpurun_out/tma_gather4.log
for E in "CC_PAIR_GATHER=1" "CC_PAIR_GATHER=0" "CC_ROWS_VARIANT=2"; do
  env $E timeout 600 python bench.py --no-cpu-baseline --no-ncu > gpurun_out/bench_pair_$E.log 2>&1; echo "$E rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_pair_$E.log').read().strip().splitlines()[-1]); print('$E', round(d['ms_per_step'],2), d['phase_ms'])"
done
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r2b.csv $CMD > gpurun_out/ncu_launch_r2b.log 2>&1; echo launch rc=$?
