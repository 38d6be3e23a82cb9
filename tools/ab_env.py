"""Same-process A/B of an environment switch on one shape: device time per factorization
and max |dR| / max|R| between the two settings.
    N=1000000 M=400 S=8 python tools/ab_env.py BGS_K2M=0"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_21791_b200 as bgs  # noqa: E402

n = int(os.environ.get("N", "1000000"))
m = int(os.environ.get("M", "400"))
s = int(os.environ.get("S", "4"))
v = int(bgs.parse_variant(os.environ.get("VARIANT", "BCGSI+P-1S")))
k, val = sys.argv[1].split("=")
ctx = bgs.Context(0)
ld = (n + 31) // 32 * 32
X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
res = {}
for setting in ("base", "alt", "base", "alt"):
    if setting == "alt":
        os.environ[k] = val
    else:
        os.environ.pop(k, None)
    ts = []
    for _ in range(4):
        r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        ts.append(tm.factor_ms)
    res.setdefault(setting, []).extend(ts)
    res[setting + "_r"] = r
    if setting == "base":
        loo, rs = bgs.metrics_device(ctx, n, m, n, X.data_ptr(), ld, Q.data_ptr(), ld, r)
        res["base_m"] = (loo, rs)
    else:
        loo, rs = bgs.metrics_device(ctx, n, m, n, X.data_ptr(), ld, Q.data_ptr(), ld, r)
        res["alt_m"] = (loo, rs)
d = np.abs(res["base_r"] - res["alt_r"]).max() / np.abs(res["base_r"]).max()
print(f"{os.environ.get('VARIANT', 'BCGSI+P-1S')} n={n} m={m} s={s}: base {np.median(res['base']):.3f} ms "
      f"(loo {res['base_m'][0]:.2e} res {res['base_m'][1]:.2e}) | {k}={val} {np.median(res['alt']):.3f} ms "
      f"(loo {res['alt_m'][0]:.2e} res {res['alt_m'][1]:.2e}) | max dR/maxR {d:.2e}")
