# Step through matgen.geometric_device at large n and check each stage.
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2507_21791_b200 as bgs
from paper_2507_21791_b200 import api, matgen
ctx = bgs.Context(0)
n, m = int(float(sys.argv[1])), 400
ld = (n + 31) // 32 * 32
x = torch.empty((m, ld), dtype=torch.float64, device="cuda")
scratch = torch.empty_like(x)
api.gen_gaussian_device(ctx, 12345, 0, n, m, scratch.data_ptr(), ld)
x.zero_()
r, st, tm = api.factor_device(ctx, 3, n, m, 4, 0, n, scratch.data_ptr(), ld, x.data_ptr(), ld)
g = (x[:, :n] @ x[:, :n].T).cpu().numpy()
print("U^T U - I max", np.abs(g - np.eye(m)).max())
vs = matgen.haar_orthogonal(m, 12345 ^ 0x5EED) * matgen.sigma_schedule(m, 1e6)[None, :]
vs_t = torch.from_numpy(np.ascontiguousarray(vs)).cuda()
torch.matmul(vs_t, x, out=scratch)
xt = scratch[:, :n]
gx = (xt @ xt.T).cpu().numpy()
ev = np.sqrt(np.sort(np.linalg.eigvalsh(gx))[::-1])
print("sv(X) head", ev[:3], "tail", ev[-3:])
y = torch.matmul(vs_t, x)
print("out= vs no out= max diff", float((y - scratch).abs().max()))
x.copy_(scratch)
q = torch.zeros_like(x)
for v in (3, 2, 1):
    r, st, tm = api.factor_device(ctx, v, n, m, 4, 0, n, x.data_ptr(), ld, q.data_ptr(), ld)
    loo, res = api.metrics_device(ctx, n, m, n, x.data_ptr(), ld, q.data_ptr(), ld, r)
    sv = np.linalg.svd(r, compute_uv=False)
    print("variant", v, "loo", loo, "res", res, "sv(R) head", sv[:3], "max rel dev from sv(X)",
          np.abs(sv / ev - 1).max())
