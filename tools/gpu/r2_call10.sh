set -x
mkdir -p gpurun_out/r2e
D=gpurun_out/r2e
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_multiproc.py -q --timeout 600 > $D/tests.log 2>&1; tail -3 $D/tests.log
DD_SETUP_TRACE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $D/bench.json 2> $D/bench.err; python -c "import json; d=json.load(open('$D/bench.json')); print(d['value'], d['apply']['ms'], d['spmv']['ms'], d['setup_ms'], d['refactor_ms'])"; grep "dd setup" $D/bench.err | head -20
