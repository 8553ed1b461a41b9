mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 $CMD > gpurun_out/plain_short.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gather_short" -c 2 -o gpurun_out/r2_short $CMD > gpurun_out/ncu_short.log 2>&1; echo rc=$?
