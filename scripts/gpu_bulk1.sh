# TMA bulk gather: parity suite, variant sweep vs the cp.async ring, launch list
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 900 python scripts/agg_sweep.py --config 3 --check --envs "CC_GATHER_IMPL=ring,bulk;CC_BULK_STAGE_BYTES=3072,6144,12288" 2>&1 | tail -12
timeout 600 python scripts/agg_sweep.py --config 2 --check --envs "CC_GATHER_IMPL=ring,bulk" 2>&1 | tail -4
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_bulk1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bulk1.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
tail -c 1500 gpurun_out/plain_bulk1.log
