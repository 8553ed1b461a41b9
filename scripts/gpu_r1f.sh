mkdir -p gpurun_out
timeout 1200 python scripts/agg_sweep.py --config 3 --envs "CC_HUB_L2_FRAC=0,0.3,0.5,0.7;CC_RING_VARIANT=0,1" 2>&1
timeout 1200 python scripts/agg_sweep.py --config 3 --envs "CC_HUB_L2_FRAC=0.5;CC_RING_VARIANT=2,3" --segs 1024,4096,16384 2>&1
