# p = 4 rows (42 vectors): lean kernel vs sub-warp rings
mkdir -p gpurun_out
for v in 4 5; do
CC_GATHER_IMPL=ring CC_RING_VARIANT=$v timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_r$v.log 2>&1 && \
CC_GATHER_IMPL=ring CC_RING_VARIANT=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo v$v rc=$?
done
