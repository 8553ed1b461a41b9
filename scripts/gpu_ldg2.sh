# lean gather (hybrid dispatch) + fused root: parity, variant sweep, launch list, ncu of the widest gather
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_LDG_VARIANT=0,1" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --precision fp64 --envs "CC_LDG_VARIANT=0,1" 2>&1 | tail -2
timeout 900 python scripts/agg_sweep.py --config 3 --envs "CC_COMBINE_IMPL=tile,lane" 2>&1 | tail -2
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_ldg2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ldg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
tail -c 700 gpurun_out/plain_ldg2.log
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD1 > gpurun_out/plain_ldg2b.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gather_ldg -s 1 -c 1 -o gpurun_out/ldg_p5 $CMD1 > gpurun_out/ncu_full_p5.log 2>&1; echo full rc=$?
tail -3 gpurun_out/ncu_full_p5.log
