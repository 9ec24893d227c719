# A/B timing of exp/*.so builds (development aid): trace counters + apply timings
mkdir -p gpurun_out
for so in ${TRACES:-}; do echo "== $so"; DD_LIB=exp/$so.so timeout 300 python tools/trace_probe.py --submods 0,16 2>&1 | grep submod; done > gpurun_out/trace_ab.log 2>&1
PROBE_LOWER=0 tools/ab_run.sh $(for s in $SOS; do echo exp/$s.so; done) > gpurun_out/ab.log 2>&1
cat gpurun_out/trace_ab.log; grep -E "==|levelset" gpurun_out/ab.log
