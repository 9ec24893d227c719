set -x
mkdir -p gpurun_out/r2i
D=gpurun_out/r2i
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "refactor or setup" > $D/t.log 2>&1; tail -2 $D/t.log
for h in 0 1 0; do
DD_HOST_ILU0=$h DD_SETUP_TRACE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_h$h.json 2> $D/bench_h$h.err; python -c "import json; d=json.load(open('$D/bench_h$h.json')); print('host_ilu0=$h', d['value'], d['setup_ms'], d['setup_phases_ms'], d['refactor_ms'])"; grep "dd setup" $D/bench_h$h.err
done
