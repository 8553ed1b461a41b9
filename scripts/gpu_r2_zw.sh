mkdir -p gpurun_out
timeout 900 python scripts/agg_sweep.py --knobs "zwarps=0,5,6,7,10,12" --reps 3 > gpurun_out/sweep_zw.log 2>&1; echo sweep rc=$?
python -c "
import json
for l in open('gpurun_out/sweep_zw.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['knobs'], d['total'], d['combine'], d['same_as_first'])"
timeout 900 python scripts/agg_sweep.py --config 2 --knobs "zwarps=0,5,7" --reps 5 > gpurun_out/sweep_zw2.log 2>&1; echo sweep2 rc=$?
python -c "
import json
for l in open('gpurun_out/sweep_zw2.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['knobs'], d['total'], d['combine'], d['same_as_first'])"
