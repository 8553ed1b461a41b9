# round-2 final evidence: smoke, full GPU suite, bench of every config, launch list + one --set full capture of configs[3]
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 3000 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu_r2z.log 2>&1; echo pytest rc=$?; tail -12 gpurun_out/pytest_gpu_r2z.log
for C in 3 2 4 1 0; do
  timeout 1500 python bench.py --config $C > gpurun_out/bench_cfg${C}_r2z.log 2>&1; echo cfg$C rc=$?; tail -c 300 gpurun_out/bench_cfg${C}_r2z.log; echo
done
timeout 600 python bench.py --config 1 --precision fp32 > gpurun_out/bench_cfg1_fp32_r2z.log 2>&1; echo cfg1fp32 rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_r2z.log 2>&1; echo ref rc=$?
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2z.csv $CMD > gpurun_out/ncu_launch_r2z.log 2>&1; echo launch rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather_ldg --launch-skip 2 --launch-count 1 -o gpurun_out/r2z_p5long $CMD > gpurun_out/ncu_full_r2z.log 2>&1; echo full rc=$?
