# split-point sweeps after the flush rewrite + ncu source capture of the p = 4 short tail
mkdir -p gpurun_out
timeout 900 python scripts/agg_sweep.py --knobs "narrow_split=-1,2,3,4" --reps 3 > gpurun_out/sweep_narrow.log 2>&1; echo sweep1 rc=$?; tail -6 gpurun_out/sweep_narrow.log
timeout 900 python scripts/agg_sweep.py --knobs "short_split=3,4,5" --reps 3 > gpurun_out/sweep_short.log 2>&1; echo sweep2 rc=$?; tail -5 gpurun_out/sweep_short.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_gather_ldg|k_gather_ring" -c 8 -o gpurun_out/r2f_gathers $CMD > gpurun_out/ncu_full_r2f.log 2>&1; echo full rc=$?; tail -2 gpurun_out/ncu_full_r2f.log
