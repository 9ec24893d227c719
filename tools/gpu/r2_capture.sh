# Round-2 final evidence: bench lines (config 3 with the CPU baseline, config 4
# both tilings, reference arm), launch list of a bench solve (host-batched loop:
# ncu cannot profile conditional-graph kernel nodes), ncu --set full of the
# apply (config 3 and config 4 with the chosen tiles), the SpMV and the direct
# ablation, the variant probe (Table 3/4 analogue), the CSR path.
set -x
D=gpurun_out/r2f
mkdir -p $D
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err
timeout 600 python bench.py --config cfg4auto --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_cfg4auto.json 2> $D/bench_cfg4auto.err
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_cfg4.json 2> $D/bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_reference.json 2> $D/bench_reference.err
DD_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $D/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $D/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_ring -s 2 -c 1 -o $D/prof_apply -f \
    python tools/ncu_target.py cfg3 3 > $D/ncu_apply.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 1 -o $D/prof_spmv -f \
    python tools/ncu_target.py cfg3 3 > $D/ncu_spmv.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_direct -s 1 -c 1 -o $D/prof_direct -f \
    python tools/ncu_target.py cfg3 3 > $D/ncu_direct.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_ring -s 2 -c 1 -o $D/prof_apply_cfg4auto -f \
    python tools/probe.py --spe10 1 --grid 60,220,85 --tiles 6,20,17 --reps 2 --solve 0 > $D/ncu_cfg4auto.log 2>&1
timeout 600 python tools/probe.py --solve 0 --reps 20 > $D/probe_cfg3.log 2>&1
timeout 900 python tools/csr_bench.py > $D/csr.jsonl 2> $D/csr.err
ls -la $D; head -c 600 $D/bench.json
