mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 python bench.py > gpurun_out/bench_r1b.log 2>&1; echo bench rc=$?
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_ring -s 1 -c 1 -o gpurun_out/gather_r1b $CMD > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
tail -2 gpurun_out/ncu_full.log
