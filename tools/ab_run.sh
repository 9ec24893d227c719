#!/bin/bash
# Time the apply of every exp/*.so (config 3) in one GPU session. Development aid.
for so in ${@:-exp/*.so}; do
  echo "== $so"
  DD_LIB=$so timeout 300 python tools/probe.py --solve 0 --reps 10 2>&1 | grep -E "^apply (levelset|direct)"
done
