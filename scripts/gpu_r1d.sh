mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 1200 python scripts/agg_sweep.py --config 3 --envs "CC_GATHER_IMPL=reg,ring;CC_RING_VARIANT=0,1,2,3" 2>&1
timeout 600 python scripts/agg_sweep.py --config 2 --envs "CC_GATHER_IMPL=reg,ring" --segs 1024,4096 2>&1
timeout 600 python scripts/agg_sweep.py --config 1 --envs "CC_GATHER_IMPL=reg,ring" --segs 1024 2>&1
