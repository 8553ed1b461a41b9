# Round 1 re-entry: parity suite, full bench line, launch list, ncu full of the gathers.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r1j.log 2>&1; echo bench rc=$?; tail -c 3000 gpurun_out/bench_r1j.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1j.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gather -c 8 -o gpurun_out/gather_r1j $CMD > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
tail -2 gpurun_out/ncu_full.log
