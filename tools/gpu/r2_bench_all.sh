# bench lines: config 3 (default), config 4 with dd_setup-chosen tiles, config 4 paper tiles
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 600 python bench.py --config cfg4auto --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4auto.json 2> gpurun_out/bench_cfg4auto.err
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
for f in gpurun_out/bench_cfg*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['iterations'], 'apply', d['apply']['ms'], d['apply']['frac_of_measured'], 'spmv', d['spmv']['ms'], 'blas1', d['blas1_ms_per_solve'], 'setup', d.get('setup_ms'), 'refactor', d.get('refactor_ms'), d['clocks'])
PY
done
