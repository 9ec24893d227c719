# final bench lines (config 3 with the CPU baseline, config 4 chosen tiles, config 5) + smoke
D=gpurun_out/r2h
mkdir -p $D
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err
timeout 600 python bench.py --config cfg4auto --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_cfg4auto.json 2> $D/bench_cfg4auto.err
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_cfg5.json 2> $D/bench_cfg5.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -n 1 $D/smoke.log
