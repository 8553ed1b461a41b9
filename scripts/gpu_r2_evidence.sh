# round-2 evidence on the current code: smoke, GPU suite, default bench,
# launch list of one configs[3] colouring, ncu --set full of the lean gathers
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2700 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r2.log 2>&1; echo bench rc=$?; tail -c 3000 gpurun_out/bench_r2.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv $CMD > gpurun_out/ncu_launch_r2.log 2>&1; echo launch rc=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_gather_ldg" -c 4 -o gpurun_out/r2_lean $CMD > gpurun_out/ncu_full_r2.log 2>&1; echo full rc=$?
tail -3 gpurun_out/ncu_full_r2.log
