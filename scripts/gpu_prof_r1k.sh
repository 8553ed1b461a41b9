# round-1 evidence: full bench line, launch list, ncu --set full of the three ldg gathers + lane combine
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r1k.log 2>&1; echo bench rc=$?; tail -c 2500 gpurun_out/bench_r1k.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_r1k.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1k.csv $CMD > gpurun_out/ncu_launch_r1k.log 2>&1; echo launch rc=$?
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD1 > gpurun_out/plain_r1k1.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_gather_ldg|k_combine_lane" -c 4 -o gpurun_out/r1k_full $CMD1 > gpurun_out/ncu_full_r1k.log 2>&1; echo full rc=$?
tail -2 gpurun_out/ncu_full_r1k.log
