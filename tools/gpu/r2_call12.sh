set -x
mkdir -p gpurun_out/r2g
D=gpurun_out/r2g
timeout 300 python -m pytest tests/test_gpu_breakdown.py -q --timeout 120 -k "rho_mid-3-1 or sigma_mid-3-1" > $D/brk.log 2>&1; grep -E "assert|Error|passed|failed" $D/brk.log | head -20
DD_HOST_ILU0=1 timeout 300 python -m pytest tests/test_gpu_breakdown.py -q --timeout 120 -k "rho_mid-3-1 or sigma_mid-3-1" > $D/brk_host.log 2>&1; tail -2 $D/brk_host.log
timeout 600 python -m pytest tests/test_gpu_edge.py -q --timeout 120 > $D/edge.log 2>&1; grep -E "assert|Error|Timeout|passed|failed" $D/edge.log | head -30
timeout 300 python - > $D/dbg.log 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle, paper_2508_04917_b200 as dd
from tests.breakdown_cases import find_case
from tests.parity import oracle_local_factors
for cat in ("rho_mid","sigma_mid"):
    c=find_case(cat,3)
    ctx=dd.dd_setup(c["rp"],c["ci"],c["v"],P=c["P"])
    f=ctx.factors(); ref=oracle_local_factors(c["S"],0,c["S"]["n"])
    for k in ("Lv","Uv","Dinv"): print(cat,k,"max|d|",np.abs(f[k]-ref[k]).max() if f[k].size else 0, f[k].size)
    r=np.random.default_rng(2).uniform(-1,1,3*c["S"]["n"])
    z=torch.empty(3*c["S"]["n"],dtype=torch.float64,device="cuda"); ctx.apply(torch.from_numpy(r).cuda(),z); torch.cuda.synchronize()
    print(cat,"apply bitwise",np.array_equal(z.cpu().numpy(),oracle.apply(c["S"],r)))
    y=torch.empty_like(z); ctx.spmv(torch.from_numpy(r).cuda(),y); torch.cuda.synchronize()
    print(cat,"spmv bitwise",np.array_equal(y.cpu().numpy(),oracle.spmv(c["S"]["rp_r"],c["S"]["ci_r"],c["S"]["v_r"],r)))
PY
cat $D/dbg.log | tail -12
