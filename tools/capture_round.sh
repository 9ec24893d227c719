#!/bin/bash
# Round evidence: bench line, ncu launch list of the bench command, ncu --set full
# of the apply (level-set, direct) and SpMV kernels. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
DD_SOLVER_VARIANT=levelset timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
DD_SOLVER_VARIANT=levelset timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_ring -s 2 -c 1 -o gpurun_out/prof_apply -f \
    python tools/ncu_target.py cfg3 3 > gpurun_out/ncu_apply.log 2>&1
DD_SOLVER_VARIANT=levelset timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 1 -o gpurun_out/prof_spmv -f \
    python tools/ncu_target.py cfg3 3 > gpurun_out/ncu_spmv.log 2>&1
DD_SOLVER_VARIANT=levelset timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_direct -s 1 -c 1 -o gpurun_out/prof_direct -f \
    python tools/ncu_target.py cfg3 3 > gpurun_out/ncu_direct.log 2>&1
ls -la gpurun_out
