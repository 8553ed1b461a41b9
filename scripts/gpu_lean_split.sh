# launch list of one configs[3] colouring with the wide-row gathers split at
# <= 32 (q = 2) and <= 8 (q = 0) neighbours: how long the short tails take
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 $CMD > gpurun_out/plain_split.log 2>&1 && \
for Q in 0 2 4; do CC_LEAN_SPLIT=$Q timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/split$Q.csv $CMD > /dev/null 2>&1; echo q$Q rc=$?; done
