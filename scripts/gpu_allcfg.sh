# every BASELINE.json config on one GPU (bench line each, with the in-run ncu
# DRAM pass for the wide configs), then the oracle's full-size times
mkdir -p gpurun_out
for C in 0 1 2 3 4; do
  timeout 1500 python bench.py --config $C > gpurun_out/bench_cfg$C.log 2>&1; echo cfg$C rc=$?
done
timeout 600 python bench.py --config 1 --precision fp32 > gpurun_out/bench_cfg1_fp32.log 2>&1; echo cfg1fp32 rc=$?
timeout 2400 python scripts/oracle_full_time.py > gpurun_out/oracle_full.log 2>&1; echo oracle rc=$?
cat gpurun_out/oracle_full.log
