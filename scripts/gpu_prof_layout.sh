# A/B of the column layout (knob layout) on the p = 5 lean gather of configs[3]: ncu of that launch
# (the 3rd neighbour-sum pass of the plan, marked by the NVTX range cc_dominant), and phase times
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ncu"
timeout 900 python scripts/agg_sweep.py --config 3 --knobs "layout=0,1,2,3" --reps 3 > gpurun_out/lay_sweep.log 2>&1; tail -4 gpurun_out/lay_sweep.log
timeout 900 $CMD > gpurun_out/plain_lay.log 2>&1 && \
for L in 0 2 3; do CC_NVTX_MARK=3 CC_LAYOUT=$L timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --nvtx --nvtx-include "cc_dominant/" -c 1 --csv --log-file gpurun_out/lay$L.csv $CMD > gpurun_out/ncu_lay$L.log 2>&1; echo lay$L rc=$?; grep -E "duration|dram__bytes|hit_rate|sectors" gpurun_out/lay$L.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'; done
