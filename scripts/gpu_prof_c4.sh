# ncu --set full: configs[4]'s fused root gather (its dominant kernel) and config 3's Z combine
mkdir -p gpurun_out
CMD4="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD4 > gpurun_out/plain_c4p.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none -k regex:k_gather_ldg -s 1 -c 1 -o gpurun_out/c4_root $CMD4 > gpurun_out/ncu_c4.log 2>&1; echo c4 rc=$?
tail -2 gpurun_out/ncu_c4.log
CMD3="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD3 > gpurun_out/plain_c3z.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_combine_z -c 1 -o gpurun_out/c3_z $CMD3 > gpurun_out/ncu_c3z.log 2>&1; echo z rc=$?
tail -2 gpurun_out/ncu_c3z.log
