# bench lines for every config on one GPU (configs[4] included)
mkdir -p gpurun_out
for c in 0 1 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_cfg$c.log 2>&1; echo cfg$c rc=$?; done
timeout 600 python bench.py --config 1 --precision fp32 --steps 10 --warmup 3 > gpurun_out/bench_cfg1_fp32.log 2>&1; echo cfg1f rc=$?
timeout 1500 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1; echo cfg4 rc=$?
for f in gpurun_out/bench_cfg*.log; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['ms_per_step'],3), round(d['value'],1), d['dtype'], round(d['roofline']['frac'] or 0,3), d['e2e']['ms_per_step'], d.get('cpu_baseline',{}).get('value'))"; done
