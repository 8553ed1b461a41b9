# round-1 final launch list (ncu gpu__time_duration, cold, serialised)
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_r1r.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1r.csv $CMD > gpurun_out/ncu_launch_r1r.log 2>&1; echo launch rc=$?
