"""Per-factorization breakdown at a given shard size (BCGSI+P-1S, m=400, s=4): device
time, the single-pass HBM floor (algorithmic bytes of the fused sweep / measured peak),
and the live profiler's per-class time and launches.  The small-shard regime is where a
GPU sits at P = 8 (n_loc = 125,000 at config 2).
    python tools/smalln_study.py 125000 100000 1000000
"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2507_21791_b200 as bgs  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6544.3
m, s = int(os.environ.get("M", "400")), int(os.environ.get("S", "4"))
v = int(bgs.parse_variant(os.environ.get("VARIANT", "BCGSI+P-1S")))
ctx = bgs.Context(0)
for n in [int(a) for a in sys.argv[1:]] or [125000]:
    ld = (n + 31) // 32 * 32
    X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
    Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
    ts = []
    for rep in range(8):
        r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        ts.append(tm.factor_ms)
    ctx.profile(True)
    bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
    prof = ctx.read_profile()
    ctx.profile(False)
    q = m // s
    alg = sum(8.0 * n * ((k + 5) * s) for k in range(1, q - 1)) + 8.0 * n * (2 * s) * 3  # ~fused sweep
    t = sorted(ts)[len(ts) // 2]
    floor = alg / (peak * 1e9) * 1e3
    print(f"n={n}: {t:.3f} ms (min {min(ts):.3f}), single-pass floor {floor:.3f} ms -> {floor / t:.3f}; "
          f"{t * 1e3 / q:.1f} us per step; launches {tm.kernel_launches}")
    for k, d in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"   {k:24s} {d['ms']:8.3f} ms  {d['launches']:4d} launches  {d['ms'] * 1e3 / max(d['launches'], 1):7.2f} us each")
    del X, Q
