# narrow-row gathers: ring variants vs lean kernel (per-launch list)
mkdir -p gpurun_out
for v in 0 2 3; do
CC_GATHER_IMPL=ring CC_RING_VARIANT=$v timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_n$v.log 2>&1 && \
CC_GATHER_IMPL=ring CC_RING_VARIANT=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo v$v rc=$?
done
