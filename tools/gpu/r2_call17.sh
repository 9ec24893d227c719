set -x
mkdir -p gpurun_out/r2k
D=gpurun_out/r2k
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_multiproc.py -q --timeout 300 -k "agreed" > $D/agree.log 2>&1; tail -3 $D/agree.log
timeout 1200 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $D/bench_cfg5.json 2> $D/bench_cfg5.err; head -c 1800 $D/bench_cfg5.json; tail -3 $D/bench_cfg5.err
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; head -c 4000 $D/bench.json
