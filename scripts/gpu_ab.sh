# A/B of two builds of libcc.so (scripts/libcc_old.so vs the tree's) on configs 2 and 3
set -e
cp paper_1804_09764_b200/libcc.so /tmp/libcc_new.so
for v in old new old new; do
  if [ $v = old ]; then cp scripts/libcc_old.so paper_1804_09764_b200/libcc.so; else cp /tmp/libcc_new.so paper_1804_09764_b200/libcc.so; fi
  for c in ${AB_CONFIGS:-2 3}; do echo "$v cfg$c $(timeout 600 python scripts/agg_sweep.py --config $c --reps 5 2>&1 | grep env | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["total"], d["gather"], d["combine"], d["csort"])')"; done
done
cp /tmp/libcc_new.so paper_1804_09764_b200/libcc.so
