set -x
mkdir -p gpurun_out/r2f
D=gpurun_out/r2f
timeout 1700 python -m pytest tests -m gpu -q --timeout 300 > $D/gputest.log 2>&1; tail -15 $D/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
for h in 0 1; do
DD_HOST_ILU0=$h DD_SETUP_TRACE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_h$h.json 2> $D/bench_h$h.err; python -c "import json; d=json.load(open('$D/bench_h$h.json')); print('host_ilu0=$h', d['value'], d['iterations'], d['apply']['ms'], d['setup_ms'], d['setup_phases_ms'], d['refactor_ms'])"; grep "dd setup" $D/bench_h$h.err | head -20
done
