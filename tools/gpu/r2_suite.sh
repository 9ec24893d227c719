# full GPU suite, smoke(), config 5 bench line
mkdir -p gpurun_out/r2s
D=gpurun_out/r2s
timeout 1500 python -m pytest tests -m gpu -x -q > $D/gputests.log 2>&1; echo "tests rc=$?"; tail -n 3 $D/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 2 $D/smoke.log
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_cfg5.json 2> $D/bench_cfg5.err; echo "cfg5 rc=$?"; head -c 700 $D/bench_cfg5.json
