# LOO / residual of P-1S on N(0,1) at large n (int-overflow hunt).
import sys
sys.path.insert(0, ".")
import torch
import paper_2507_21791_b200 as bgs
ctx = bgs.Context(0)
m, s = 400, 4
for n in [int(float(a)) for a in sys.argv[1:]]:
    ld = (n + 31) // 32 * 32
    X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
    Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
    for env in [None]:
        r, st, tm = bgs.factor_device(ctx, 3, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        loo, res = bgs.metrics_device(ctx, n, m, n, X.data_ptr(), ld, Q.data_ptr(), ld, r)
        qn = torch.linalg.vector_norm(Q[:, :n], dim=1)
        print(f"n={n:.1e} loo={loo:.3e} res={res:.3e} colnorm-1 max={float((qn - 1).abs().max()):.3e} "
              f"ms={tm.factor_ms:.1f}", flush=True)
    del X, Q
    torch.cuda.empty_cache()
