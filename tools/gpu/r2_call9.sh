# round-2 GPU call 9: setup timing after the host-side changes, refactor /
# setup parity tests, sanitizer runs (graph vs batched loop, two contexts)
set -x
mkdir -p gpurun_out/r2d
D=gpurun_out/r2d
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py -q --timeout 600 > $D/parity.log 2>&1; tail -3 $D/parity.log
DD_SETUP_TRACE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $D/bench.json 2> $D/bench.err; python -c "import json; d=json.load(open('$D/bench.json')); print(d['value'], d['apply']['ms'], d['setup_ms'], d['refactor_ms'])"; grep "dd setup" $D/bench.err | head -20
SAN_WORLD2=0 SAN_CASES=1,2 DD_GRAPH=0 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_target.py > $D/memcheck_batched.log 2>&1; tail -3 $D/memcheck_batched.log
SAN_WORLD2=0 SAN_CASES=1,2 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_target.py > $D/memcheck_graph.log 2>&1; tail -3 $D/memcheck_graph.log
SAN_WORLD2=0 SAN_CASES=2 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_target.py > $D/memcheck_graph_single.log 2>&1; tail -3 $D/memcheck_graph_single.log
SAN_WORLD2=0 SAN_CASES=1,2 CUDA_LAUNCH_BLOCKING=1 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_target.py > $D/memcheck_graph_blocking.log 2>&1; tail -3 $D/memcheck_graph_blocking.log
