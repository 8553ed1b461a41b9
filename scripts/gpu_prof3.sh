mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_ring -s 1 -c 1 -o gpurun_out/gather_r1c $CMD > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
tail -2 gpurun_out/ncu_full.log
