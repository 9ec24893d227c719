# round-2 GPU call 8: refactor kernel A/B (parity + time), full GPU suite,
# smoke, default bench
set -x
mkdir -p gpurun_out/r2c
D=gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "refactor" > $D/refactor_tests.log 2>&1; tail -3 $D/refactor_tests.log
for k in 1 2; do
DD_REFACTOR_KERNEL=$k timeout 600 python -c "
import sys,time; sys.path.insert(0,'.')
import torch, paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3
rp,ci,v=laplacian_bsr3(160,160,160)
c=dd.dd_setup(rp,ci,v,grid=(160,160,160),tiles=(16,16,8),enable_refactor=True)
vd=torch.from_numpy(v).cuda(); c.refactor(vd); torch.cuda.synchronize()
t=time.time(); [c.refactor(vd) for _ in range(5)]; torch.cuda.synchronize(); print('kernel $k refactor ms', (time.time()-t)*200)
"
done
timeout 1700 python -m pytest tests -m gpu -q --timeout 300 > $D/gputest.log 2>&1; tail -4 $D/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; head -c 3000 $D/bench.json
