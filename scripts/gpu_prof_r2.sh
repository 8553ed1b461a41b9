# round-2 evidence: launch list of one configs[3] colouring + ncu --set full of
# the narrow gathers, the Z-block combine and the p = 5 lean gather
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 $CMD > gpurun_out/plain_r2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv $CMD > gpurun_out/ncu_launch_r2.log 2>&1; echo launch rc=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_gather_rows|k_gather_ring|k_combine_z|k_csort" -c 8 -o gpurun_out/r2_narrow $CMD > gpurun_out/ncu_full_r2.log 2>&1; echo full rc=$?
tail -3 gpurun_out/ncu_full_r2.log
