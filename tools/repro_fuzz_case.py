import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_21791_b200 as bgs
from oracle.oracle import Oracle
o = Oracle()
v, n, m, s, kappa, gauss, seed = 5, 49, 12, 4, 1280.7671752796468, False, 343794
x = o.gen_matrix(n, m, s, kappa, seed, gauss)
ref = o.factor(v, x, s, 1, metrics=True)
print("oracle loo %.2e res %.2e" % (ref.loo, ref.resid))
for P in (1, 2, 3):
    r2 = o.factor(v, x, s, P, metrics=True); print("oracle P=%d loo %.2e" % (P, r2.loo))
out = bgs.run_factor(v, x, s, 1, metrics=False, ctx=bgs.Context(0))
print("bgs_factor loo %.2e  dR %.1e" % (o.loo(out.q), np.abs(out.r-ref.r).max()/np.abs(ref.r).max()))
ctx = bgs.Context(0, 0, 1, bgs.nccl_unique_id())
ld = 64
X = torch.zeros((m, ld), dtype=torch.float64, device="cuda"); X[:, :n] = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
Q = torch.zeros_like(X)
r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
q = np.asfortranarray(Q[:, :n].cpu().numpy().T)
print("factor_device(nccl) loo %.2e dR %.1e" % (o.loo(q), np.abs(r-ref.r).max()/np.abs(ref.r).max()))
for seed2 in range(5):
    x2 = o.gen_matrix(n, m, s, kappa, seed + 1 + seed2, gauss); rr = o.factor(v, x2, s, 1, metrics=True)
    oo = bgs.run_factor(v, x2, s, 1, metrics=False, ctx=bgs.Context(0))
    print("nearby seed oracle %.2e gpu %.2e" % (rr.loo, o.loo(oo.q)))
