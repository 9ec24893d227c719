set -x
mkdir -p gpurun_out/r2m
D=gpurun_out/r2m
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q --timeout 300 -k "fused" > $D/fused.log 2>&1; tail -3 $D/fused.log
timeout 1500 python tools/ablation_stats.py > $D/ablation_stats.jsonl 2> $D/ablation_stats.err; cat $D/ablation_stats.jsonl; tail -3 $D/ablation_stats.err
