mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "short_list or knob or twins or small_suite or loopback or config0 or config1 or sibling" > gpurun_out/pytest_ring.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ring.log
timeout 600 python scripts/agg_sweep.py --knobs "combine_wreg=1,0" --reps 3 > gpurun_out/sweep_ring.log 2>&1; echo sweep rc=$?; tail -2 gpurun_out/sweep_ring.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2m.csv $CMD > gpurun_out/ncu_launch_r2m.log 2>&1; echo launch rc=$?
python scripts/launches_table.py gpurun_out/launches_r2m.csv 2>/dev/null | head -16 | cut -c1-200
