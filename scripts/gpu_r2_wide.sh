mkdir -p gpurun_out
timeout 1500 python scripts/agg_sweep.py --config 4 --knobs "wide_warps=0,6,4;wide_nv=4,6" --reps 1 > gpurun_out/sweep_wide.log 2>&1; echo sweep rc=$?
python -c "
import json
for l in open('gpurun_out/sweep_wide.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['knobs'], d['total'], d['gather'], d['combine'], d['same_as_first'])"
CMD="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch_c4.log 2>&1; echo launch rc=$?
python scripts/launches_table.py gpurun_out/launches_c4.csv 2>/dev/null | cut -c1-180 | head -30
