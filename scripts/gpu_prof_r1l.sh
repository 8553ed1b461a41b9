# evidence after the Z combine: full bench line, launch list, ncu --set full of the dominant gather + Z combine
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r1l.log 2>&1; echo bench rc=$?; tail -c 3000 gpurun_out/bench_r1l.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_r1l.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1l.csv $CMD > gpurun_out/ncu_launch_r1l.log 2>&1; echo launch rc=$?
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD1 > gpurun_out/plain_r1l1.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_gather_ldg|k_combine_z" -c 3 -o gpurun_out/r1l_full $CMD1 > gpurun_out/ncu_full_r1l.log 2>&1; echo full rc=$?
tail -2 gpurun_out/ncu_full_r1l.log
