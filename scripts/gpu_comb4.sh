# combine: shared split table + single-IMAD addressing; intensity switch
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_COMBINE_V=1,2" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --precision fp64 --check --envs "CC_COMBINE_V=1,2" 2>&1 | tail -2
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_comb4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_comb4.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
tail -c 600 gpurun_out/plain_comb4.log
