# round-2 GPU call 3: the GPU suite (no -x), swizzle A/B at cfg3, the paper's
# variants (Table 3/4 analogue), cfg4 vs automatic tiles, ncu bank conflicts
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gputest3.log 2>&1; tail -15 gpurun_out/gputest3.log
for swz in 1 0; do
  DD_SWZ=$swz timeout 600 python tools/probe.py --reps 20 --solve 1 > gpurun_out/probe_cfg3_swz$swz.log 2>&1
  grep -E "tiles|apply|spmv|bicgstab" gpurun_out/probe_cfg3_swz$swz.log | cut -c1-200
done
PROBE_LOWER=0 timeout 600 python tools/probe.py --spe10 1 --grid 60,220,85 --tiles 10,20,17 --reps 20 > gpurun_out/probe_cfg4.log 2>&1
PROBE_LOWER=0 timeout 600 python tools/probe.py --spe10 1 --grid 60,220,85 --tiles auto --reps 20 > gpurun_out/probe_cfg4auto.log 2>&1
grep -E "tiles|apply levelset|apply direct |bicgstab" gpurun_out/probe_cfg4*.log | cut -c1-220
for swz in 1 0; do
  DD_SWZ=$swz timeout 600 ncu --clock-control none -k regex:k_apply_ring -s 2 -c 1 \
    --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    python tools/probe.py --reps 2 --solve 0 > gpurun_out/ncu_swz$swz.log 2>&1
  grep -E "k_apply_ring|duration|bank|wavefronts|dram__bytes" gpurun_out/ncu_swz$swz.log | head -8
done
