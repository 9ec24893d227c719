# round-2 GPU call 6: ncu captures for profiles/ (apply cfg3, SpMV, direct,
# edge, ilu0, cfg4 both tilings), launch list (batched loop: ncu cannot
# profile kernel nodes of conditional graphs), bench lines cfg3 / cfg4auto
set -x
mkdir -p gpurun_out/r2
D=gpurun_out/r2
P="python tools/probe.py --reps 2 --solve 0"
PROBE_VARS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_ring -s 2 -c 1 -o $D/prof_apply -f $P > $D/p1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv -s 3 -c 1 -o $D/prof_spmv -f $P > $D/p2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_direct -s 2 -c 1 -o $D/prof_direct -f $P > $D/p3.log 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:k_apply_ring<3, 65536u, 16384u, false, 0, 1>" -s 2 -c 1 -o $D/prof_edge -f $P > $D/p4.log 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:k_apply_ring<3, 65536u, 16384u, false, 0, 2>" -s 2 -c 1 -o $D/prof_ilu0 -f $P > $D/p5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_ring -s 2 -c 1 -o $D/prof_apply_cfg4auto -f python tools/probe.py --spe10 1 --grid 60,220,85 --tiles 6,20,17 --reps 2 --solve 0 > $D/p6.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_apply_ring -s 2 -c 1 -o $D/prof_apply_cfg4 -f python tools/probe.py --spe10 1 --grid 60,220,85 --tiles 10,20,17 --reps 2 --solve 0 > $D/p7.log 2>&1
DD_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $D/launches.out 2>&1
ls -la $D
timeout 600 python bench.py --config cfg4auto --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_cfg4auto.json 2> $D/bench_cfg4auto.err; head -c 1500 $D/bench_cfg4auto.json
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_cfg4.json 2> $D/bench_cfg4.err; head -c 600 $D/bench_cfg4.json
