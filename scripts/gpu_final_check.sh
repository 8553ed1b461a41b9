# driver-like round-end check: full GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q --durations=6 2>&1 | tail -12
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/bench_final.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -c 600 gpurun_out/bench_ref.log
