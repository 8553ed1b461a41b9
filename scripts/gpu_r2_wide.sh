# configs[4]'s fused-root p = 7 gather (13.7 KB N'' rows) on the scale-20 twin: wide-row knob sweep
mkdir -p gpurun_out
for ww in 0 4 2; do for nv in 4 6; do
  CC_WIDE_WARPS=$ww CC_WIDE_NV=$nv timeout 600 python scripts/prof_c4_combine.py 20 64 3 > gpurun_out/wide_w${ww}_nv${nv}.log 2>&1
  echo "wide_warps=$ww wide_nv=$nv rc=$? $(tail -1 gpurun_out/wide_w${ww}_nv${nv}.log | grep -o "'gather': [0-9.]*")"
done; done
