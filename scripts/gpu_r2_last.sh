# last check of the final defaults: smoke, parity subset, default bench (configs[3]), configs[2] bench
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "not full" > gpurun_out/pytest_last.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_last.log
timeout 900 python bench.py > gpurun_out/bench_cfg3_r2last.log 2>&1; echo bench rc=$?; tail -c 600 gpurun_out/bench_cfg3_r2last.log; echo
timeout 600 python bench.py --config 2 > gpurun_out/bench_cfg2_r2last.log 2>&1; echo bench2 rc=$?
