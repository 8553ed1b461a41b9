# configs[4]'s (7;4,3) combine: global-table Z-block kernel vs the lane kernel; parity of the k = 15 shapes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "twins or knob_setting or static_cover" > gpurun_out/pytest_zg.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_zg.log
for zg in 1 0; do CC_COMBINE_ZGLOBAL=$zg timeout 600 python scripts/prof_c4_combine.py 20 64 3 > gpurun_out/c4comb_zg$zg.log 2>&1; echo zg=$zg rc=$?; tail -1 gpurun_out/c4comb_zg$zg.log; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_combine_z" -c 1 -o gpurun_out/r2_c4zg python scripts/prof_c4_combine.py 20 64 1 > gpurun_out/ncu_c4zg.log 2>&1; echo full rc=$?; tail -2 gpurun_out/ncu_c4zg.log
