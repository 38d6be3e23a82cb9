import sys, os
sys.path.insert(0, ".")
import torch
import paper_2507_21791_b200 as bgs
ctx = bgs.Context(0)
n, m, s = 1000000, 800, 4
v = int(bgs.parse_variant("BCGSI+P-1S"))
ld = (n + 31) // 32 * 32
X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
Q = torch.empty((m, ld), dtype=torch.float64, device="cuda")
bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
for rep in range(3):
    r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
    print("m=800", os.environ.get("BGS_K12C_PLAN_MAXC", ""), tm.factor_ms, "ms", tm.kernel_launches, "launches")
print(bgs.metrics_device(ctx, n, m, n, X.data_ptr(), ld, Q.data_ptr(), ld, r))
