#!/bin/bash
# (ncu captures: DD_SOLVER_VARIANT=levelset skips the setup-time variant timing, so -s/-c count only the target launches)
# spin-loop (Alg. 4) vs level-set (Alg. 6) vs direct at
# 64^3 with P 2048 (2a) and P 8192 (2b): CUDA-event timings (L2 flushed and
# warm) and one ncu --set full capture per variant. Outputs under gpurun_out/.
mkdir -p gpurun_out
for c in 2a 2b; do
  tiles=16,16,8; [ $c = 2b ] && tiles=32,16,16
  timeout 300 python tools/probe.py --grid 64,64,64 --tiles $tiles --solve 0 --reps 30 > gpurun_out/cfg${c}_probe.log 2>&1
  timeout 300 python tools/probe.py --grid 64,64,64 --tiles $tiles --solve 0 --reps 30 --warm 1 > gpurun_out/cfg${c}_probe_warm.log 2>&1
  for v in levelset spin direct; do
    DD_SOLVER_VARIANT=levelset timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 \
      -o gpurun_out/cfg${c}_$v -f python tools/ncu_target.py cfg$c 3 $v > gpurun_out/cfg${c}_${v}_ncu.log 2>&1
  done
done
ls gpurun_out
