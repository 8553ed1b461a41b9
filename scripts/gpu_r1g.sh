mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 1200 python scripts/agg_sweep.py --config 3 --envs "CC_HUB_L2_FRAC=0.5,0.7;CC_RING_VARIANT=0,1" --fixed-root 0,1 2>&1
timeout 1200 python scripts/agg_sweep.py --config 2 --envs "CC_HUB_L2_FRAC=0.5" --segs 1024 --fixed-root 0,1 2>&1
