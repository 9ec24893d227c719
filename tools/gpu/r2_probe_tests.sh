# round-2 GPU call: probes (cross-process IPC ping-pong, NCCL two ranks on one
# GPU), the GPU test suite, a default bench line
set -x
mkdir -p gpurun_out
nvidia-smi -L; which nvidia-cuda-mps-control; nproc; lscpu | grep -i "model name"
d=$(mktemp -d)
timeout 60 tools/micro/ipc_pingpong server $d 2000 > gpurun_out/pp_server.log 2>&1 &
sp=$!
timeout 60 tools/micro/ipc_pingpong client $d 2000 > gpurun_out/pp_client.log 2>&1
wait $sp
cat gpurun_out/pp_*.log
timeout 120 python tools/micro/nccl_dup_probe.py > gpurun_out/nccl_dup.log 2>&1; tail -5 gpurun_out/nccl_dup.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gputest.log 2>&1; tail -30 gpurun_out/gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; head -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
