# quick A/B of a kernel change: parity subset, configs[3] phases (3 reps), launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "short_list or every_knob or twins or config1 or small_suite or fused_root or sibling or determinism" > gpurun_out/pytest_ab.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_ab.log
timeout 1200 python scripts/agg_sweep.py --config 3 --knobs "${KNOBS:-fused_root=1}" --check --reps 3 > gpurun_out/sweep_ab_c3.log 2>&1; echo sweep rc=$?; tail -6 gpurun_out/sweep_ab_c3.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_ab.csv $CMD > gpurun_out/ncu_launch_ab.log 2>&1; echo launch rc=$?
python scripts/launches_table.py gpurun_out/launches_ab.csv 2>&1 | tail -17
