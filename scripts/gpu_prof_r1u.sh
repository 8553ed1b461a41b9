# final round-1 evidence: launch list + ncu --set full of the dominant gather (p = 5) alone
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_r1u.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1u.csv $CMD > gpurun_out/ncu_launch_r1u.log 2>&1; echo launch rc=$?
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 $CMD1 > gpurun_out/plain_r1u1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gather_ldg -s 1 -c 1 -o gpurun_out/r1u_p5 $CMD1 > gpurun_out/ncu_full_r1u.log 2>&1; echo full rc=$?
tail -2 gpurun_out/ncu_full_r1u.log
