mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 900 python scripts/agg_sweep.py --config 2 --variants 0,1,2,3,4 --segs 512,4096 2>&1
timeout 1200 python scripts/agg_sweep.py --config 3 --variants 0,1,2,4 --segs 4096 2>&1
