# round-2 (session 5) evidence at HEAD: smoke, full GPU suite, default bench, launch list of configs[3]
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 3000 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu_r2s5.log 2>&1; echo pytest rc=$?; tail -12 gpurun_out/pytest_gpu_r2s5.log
timeout 900 python bench.py > gpurun_out/bench_cfg3_r2s5.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/bench_cfg3_r2s5.log; echo
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2s5.csv $CMD > gpurun_out/ncu_launch_r2s5.log 2>&1; echo launch rc=$?
