# driver-like evidence on the current code: smoke, GPU suite, bench (ours + reference arm),
# launch list with DRAM bytes, ncu --set full of the p = 5 gather launches
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 3000 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_final.log 2>&1; echo pytest rc=$?; tail -9 gpurun_out/pytest_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?; tail -c 600 gpurun_out/bench_final.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1; echo ref rc=$?; tail -c 300 gpurun_out/bench_ref_final.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2final.csv $CMD > gpurun_out/ncu_launch_final.log 2>&1; echo launch rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_gather_ldg<float, 3" -c 2 -o gpurun_out/r2final_p5 $CMD > gpurun_out/ncu_full_final.log 2>&1; echo full rc=$?
