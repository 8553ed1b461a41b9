# ncu --set full with source correlation of the Z-block combine (+ fused root) on config 3
mkdir -p gpurun_out
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD1 > gpurun_out/plain_src.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_combine_z -c 1 -o gpurun_out/src_z $CMD1 > gpurun_out/ncu_src_z.log 2>&1; echo full rc=$?
tail -1 gpurun_out/ncu_src_z.log
