# lean gather: branch-free flush + map-derived vector skip; parity subset, bench A/B, launch list
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x -k "short_list or knob or twins or config0 or small_suite or fused or config1 or sibling or heavy" > gpurun_out/pytest_flush2.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_flush.log
for E in "CC_SHORT_LISTS=2" "CC_NARROW_IMPL=0"; do
  env $E timeout 600 python bench.py --no-cpu-baseline --no-ncu > gpurun_out/bench_flush2_$E.log 2>&1; echo "$E rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_flush2_$E.log').read().strip().splitlines()[-1]); print('$E', round(d['ms_per_step'],2), d['phase_ms'])"
done
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2e.csv $CMD > gpurun_out/ncu_launch_r2e.log 2>&1; echo launch rc=$?
python scripts/launches_table.py gpurun_out/launches_r2e.csv | head -16 | cut -c1-200
