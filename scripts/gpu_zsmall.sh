# small combines through the Z kernel vs the V-tile kernel
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/p0.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_z0.csv $CMD > /dev/null 2>&1; echo a rc=$?
CC_COMBINE_Z_SMALL=1 timeout 600 $CMD > gpurun_out/p1.log 2>&1 && CC_COMBINE_Z_SMALL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_z1.csv $CMD > /dev/null 2>&1; echo b rc=$?
CC_COMBINE_Z_SMALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_suite or config1 or twins" 2>&1 | tail -2
