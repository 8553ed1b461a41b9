# compile-time-cover combine (combine_s.cu): parity, A/B against the run-time cover, launch list, ncu of the kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "static_cover or fused_combine or knob_setting or twins_fp32 or config3_full" > gpurun_out/pytest_static.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_static.log
for cfg in 3 2; do for st in 1 0; do
  CC_COMBINE_STATIC=$st timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-ncu > gpurun_out/bench_static_c${cfg}_s${st}.log 2>&1
  echo "cfg=$cfg static=$st rc=$?"; python -c "import json,sys; d=json.loads(open('gpurun_out/bench_static_c${cfg}_s${st}.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phase_ms'])"
done; done
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_r2s.csv $CMD > gpurun_out/ncu_launch_s.log 2>&1; echo launch rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_combine_s" -c 1 -o gpurun_out/r2s_combine $CMD > gpurun_out/ncu_full_s.log 2>&1; echo full rc=$?
