mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "short_list or knob or fused or twins" > gpurun_out/pytest_zp.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_zp.log
timeout 900 python scripts/agg_sweep.py --knobs "zparam=0,1;short_lists=2,5" --reps 3 > gpurun_out/sweep_zp.log 2>&1; echo sweep rc=$?; tail -4 gpurun_out/sweep_zp.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
CC_SHORT_LISTS=5 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2i.csv $CMD > gpurun_out/ncu_launch_r2i.log 2>&1; echo launch rc=$?
python scripts/launches_table.py gpurun_out/launches_r2i.csv 2>/dev/null | head -16 | cut -c1-200
