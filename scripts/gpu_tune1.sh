# gather: L2 prefetch variant x L2 persistence window; ncu of the lane combine
mkdir -p gpurun_out
timeout 1500 python scripts/agg_sweep.py --config 3 --check --envs "CC_LDG_VARIANT=0,3;CC_L2_PERSIST_MB=0,64,96" 2>&1 | tail -6
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD1 > gpurun_out/plain_tune1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_combine_lane -s 2 -c 1 -o gpurun_out/comb_lane $CMD1 > gpurun_out/ncu_comb.log 2>&1; echo full rc=$?
tail -2 gpurun_out/ncu_comb.log
