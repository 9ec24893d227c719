# round-2 GPU call 4: the GPU suite (no -x, per-test timeout), smoke, bench,
# memcheck of the graph solve with two contexts
set -x
mkdir -p gpurun_out
export DD_PEER_TIMEOUT_S=60
timeout 1700 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/gputest4.log 2>&1; tail -25 gpurun_out/gputest4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1; tail -3 gpurun_out/smoke4.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; head -c 2500 gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
SAN_WORLD2=0 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_target.py > gpurun_out/memcheck4.log 2>&1; tail -8 gpurun_out/memcheck4.log
