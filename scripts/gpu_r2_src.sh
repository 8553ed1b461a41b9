# ncu --set full with source of one lean-gather launch of configs[3] (SKIP = index among the k_gather_ldg launches: 1 = p=4 short tail, 3 = p=5 short tail)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"${KERN:-k_gather_ldg}" --launch-skip ${SKIP:-3} --launch-count 1 -o gpurun_out/r2_src_${TAG:-tail5} $CMD > gpurun_out/ncu_src.log 2>&1; echo full rc=$?; tail -3 gpurun_out/ncu_src.log; ls -la gpurun_out/*.ncu-rep
