#!/bin/bash
# bench (no CPU baseline) for every exp/*.so: solve ms, in-solve SpMV/apply ms. Development aid.
for so in ${@:-exp/*.so}; do
  DD_LIB=$so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$so', 'solve', d['value'], 'spmv', d['spmv']['ms'], 'apply', d['apply']['ms'], 'blas1', d['blas1_ms_per_solve'])"
done
