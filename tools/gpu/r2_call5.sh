# round-2 GPU call 5: swizzle A/B inside the timed solves, cfg4 tilings,
# ncu --set full of the level-set apply (source-level), launch list
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ring.py -q --timeout 200 > gpurun_out/ring5.log 2>&1; tail -3 gpurun_out/ring5.log
for swz in 0 1; do
  DD_SWZ=$swz timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench5_swz$swz.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench5_swz$swz.json')); print('swz $swz', d['value'], d['apply']['ms'], d['apply']['launch'], d['spmv']['ms'], d['blas1_ms_per_solve'])"
done
for t in 10,20,17 6,20,17 12,22,17; do
  PROBE_LOWER=0 timeout 600 python tools/probe.py --spe10 1 --grid 60,220,85 --tiles $t --reps 20 > gpurun_out/probe5_cfg4_$t.log 2>&1
  grep -E "tiles|apply levelset|bicgstab" gpurun_out/probe5_cfg4_$t.log | cut -c1-230
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_ring -s 2 -c 1 -o gpurun_out/ncu5_apply_full -f \
  python tools/probe.py --reps 2 --solve 0 > gpurun_out/ncu5_full.log 2>&1; tail -3 gpurun_out/ncu5_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/launches5.out 2>&1; tail -2 gpurun_out/launches5.out
