"""One (or a few) factorizations at a given shape on cuda:0 -- a target for ncu captures.
    N=1000000 M=400 S=8 VARIANT=BCGSI+P-1S REPS=1 python tools/one_factor.py"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2507_21791_b200 as bgs  # noqa: E402

n = int(os.environ.get("N", "1000000"))
m = int(os.environ.get("M", "400"))
s = int(os.environ.get("S", "4"))
v = int(bgs.parse_variant(os.environ.get("VARIANT", "BCGSI+P-1S")))
ctx = bgs.Context(0)
ld = (n + 31) // 32 * 32
X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
for _ in range(int(os.environ.get("REPS", "1"))):
    r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
    print(f"{tm.factor_ms:.3f} ms, {tm.kernel_launches} launches")
