# full GPU suite + default bench (driver-like) + launch list
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_full.log 2>&1; echo pytest rc=$?; tail -18 gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/bench_full.log
