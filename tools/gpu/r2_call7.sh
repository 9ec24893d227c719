# round-2 GPU call 7: refactor parity + timing, ablation table at cfg3,
# ncu of the ablation kernels and of k_refactor
set -x
mkdir -p gpurun_out/r2b
D=gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "refactor" > $D/refactor_tests.log 2>&1; tail -3 $D/refactor_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > $D/bench.json 2> $D/bench.err; python -c "import json; d=json.load(open('$D/bench.json')); print(d['value'], d['apply']['ms'], d['refactor_ms'], d['setup_ms'], d['levels_device_ms'])"
timeout 900 python tools/probe.py --reps 20 --solve 0 > $D/probe_cfg3.log 2>&1; grep -E "tiles|apply|spmv" $D/probe_cfg3.log | cut -c1-170
for kv in "0, 0, 1>:edge" "0, 0, 2>:ilu0" "0, 0, 3>:tree"; do
  k=${kv%%:*}; n=${kv##*:}
  timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:k_apply_ring<3, 65536, 16384, $k" -s 2 -c 1 -o $D/prof_$n -f python tools/probe.py --reps 2 --solve 0 > $D/ncu_$n.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:k_refactor -c 1 -o $D/prof_refactor -f python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3
rp,ci,v=laplacian_bsr3(160,160,160)
c=dd.dd_setup(rp,ci,v,grid=(160,160,160),tiles=(16,16,8),enable_refactor=True)
c.refactor(torch.from_numpy(v).cuda()); torch.cuda.synchronize()
" > $D/ncu_refactor.log 2>&1; tail -2 $D/ncu_refactor.log
ls -la $D
