# Two different matrices of one shape through bgs_factor_device with the same buffers: the second
# call captures a CUDA graph.  python tools/repro_graph2.py [nccl|local]
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_21791_b200 as bgs
from oracle.oracle import Oracle
o = Oracle()
v, n, m, s = 1, 56, 54, 6
A = o.gen_matrix(n, m, s, 79816.2588371988, 755161, False)
B = o.gen_matrix(n, m, s, 2.7011009494408684, 234819, True)
ctx = bgs.Context(0, 0, 1, bgs.nccl_unique_id()) if (sys.argv[1:] or ["nccl"])[0] == "nccl" else bgs.Context(0)
ld = 64
X = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
for name, x in [("A", A), ("B", B), ("B", B), ("A", A), ("B", B)]:
    X.zero_(); Q.zero_()
    X[:, :n] = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(x).T)).cuda()
    ref = o.factor(v, x, s, 1, metrics=True)
    try:
        r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        q = np.asfortranarray(Q[:, :n].cpu().numpy().T)
        print(name, "ok loo %.2e (oracle %.2e) dR %.1e launches %d" % (o.loo(q), ref.loo, np.abs(r - ref.r).max() / np.abs(ref.r).max(), tm.kernel_launches))
    except Exception as e:
        print(name, "EXC", str(e)[:120])
