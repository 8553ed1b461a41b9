# configs[4]'s (7;4,3) combine on a scale-20 twin: phase times, then ncu --set full of the combine kernel
mkdir -p gpurun_out
timeout 600 python scripts/prof_c4_combine.py 20 64 3 > gpurun_out/c4comb_times.log 2>&1; echo rc=$?; tail -3 gpurun_out/c4comb_times.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_combine_z" -c 1 -o gpurun_out/r2_c4comb python scripts/prof_c4_combine.py 20 64 1 > gpurun_out/ncu_c4comb.log 2>&1; echo full rc=$?; tail -3 gpurun_out/ncu_c4comb.log
