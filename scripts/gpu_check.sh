set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 900 python bench.py --steps 3 --warmup 2 --config 1 --no-cpu-baseline 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 2 --config 2 --no-cpu-baseline 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 3 2>&1 | tail -3
