# GPU suite + default bench (the driver's round-end checks), logs under gpurun_out/
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2700 python -m pytest tests -m gpu -q -x --durations=8 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -c 2500 gpurun_out/bench.log
fi
