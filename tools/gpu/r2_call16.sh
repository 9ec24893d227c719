set -x
mkdir -p gpurun_out/r2j
D=gpurun_out/r2j
timeout 2000 python -m pytest tests -m gpu -q --timeout 300 > $D/gputest.log 2>&1; tail -5 $D/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
for h in 0 1 0 1; do
DD_HOST_ILU0=$h timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_h$h.json 2> $D/bench_h$h.err; python -c "import json; d=json.load(open('$D/bench_h$h.json')); print('host_ilu0=$h', d['value'], d['setup_ms'], d['setup_phases_ms'], d['refactor_ms'])"
done
