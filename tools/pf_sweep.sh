#!/bin/bash
# L2-prefetch distance sweep for the direct apply (config 3). Development aid.
out=${1:-gpurun_out/pf_sweep.txt}
mkdir -p gpurun_out; : > $out
for kb in 0 16 32 64 96 128 192 256 384; do
  echo "PF_KB=$kb" >> $out
  DD_DIRECT_PF_KB=$kb timeout 300 python tools/probe.py --solve 0 --reps 10 2>&1 | grep -E "^apply direct" >> $out
done
