mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "short_list or knob" > gpurun_out/pytest_ldg2.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ldg2.log
timeout 900 python scripts/agg_sweep.py --knobs "short_lists=2,5,6" --reps 3 > gpurun_out/sweep_ldg2.log 2>&1; echo sweep rc=$?; tail -3 gpurun_out/sweep_ldg2.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
CC_SHORT_LISTS=5 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2h.csv $CMD > gpurun_out/ncu_launch_r2h.log 2>&1; echo launch rc=$?
python scripts/launches_table.py gpurun_out/launches_r2h.csv 2>/dev/null | head -16 | cut -c1-200
