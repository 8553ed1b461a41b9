# narrow-row gathers: default vs smaller rings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for v in 0 2 3; do
CC_RING_VARIANT=$v timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_m$v.log 2>&1 && \
CC_RING_VARIANT=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_m$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo v$v rc=$?
done
