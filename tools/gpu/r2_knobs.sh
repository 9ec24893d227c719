SOS="cur ch8 pf16 pf64 cur" bash tools/gpu/call_ab.sh
echo "== DD_SWZ=0 cur"; DD_SWZ=0 DD_LIB=exp/cur.so PROBE_LOWER=0 timeout 300 python tools/probe.py --solve 0 --reps 10 2>&1 | grep -E "^apply levelset"
echo "== DD_APPLY_MODE=1 cur (streaming ceiling)"; DD_APPLY_MODE=1 DD_LIB=exp/cur.so PROBE_LOWER=0 timeout 300 python tools/probe.py --solve 0 --reps 10 2>&1 | grep -E "^apply levelset"
