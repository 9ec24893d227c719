import sys, os; sys.path.insert(0,'.')
import numpy as np, torch, oracle, paper_2508_04917_b200 as dd
from tests.breakdown_cases import find_case
c=find_case("rho_mid",3)
rp,ci,v,P=c["rp"],c["ci"],c["v"],c["P"]
print("n",rp.shape[0]-1,"P",P)
r=np.random.default_rng(2).uniform(-1,1,3*(rp.shape[0]-1))
zref=oracle.apply(c["S"],r)
def run(ctx,var=dd.DD_LEVELSET):
    z=torch.zeros(r.size,dtype=torch.float64,device="cuda"); ctx.apply(torch.from_numpy(r).cuda(),z,var); torch.cuda.synchronize(); return z.cpu().numpy()
os.environ["DD_HOST_ILU0"]="0"
g=dd.dd_setup(rp,ci,v,P=P, variants=7)
for var in (1,2,4): 
    zg=run(g,var); print("gpu-path var",var,"bitwise",np.array_equal(zg,zref),"maxdiff",np.abs(zg-zref).max())
print("zref",zref[:6]); print("zgpu",run(g)[:6])
S=c["S"]; print("oracle dinv row0", S["dinv"][:9])
print("gpu dinv row0", g.factors()["Dinv"][:9])
