mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 1200 python scripts/agg_sweep.py --config 3 --variants 0,1,2,3,4 --segs 4096 2>&1
timeout 600 python scripts/agg_sweep.py --config 2 --variants 0,1 --segs 1024,4096 2>&1
