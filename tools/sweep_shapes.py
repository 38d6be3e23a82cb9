# Functional + timing sweep over BASELINE configs 3-4 shapes on one GPU: every variant, s in
# {1,2,4,8,16} at n=1e6 m=400, and s=4 at m in {100,200,400,800} / n in {1e5,1e6,4e6}.
# Prints ms per factorization (device) or the error; verifies LOO/residual on the device.
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2507_21791_b200 as bgs

NAMES = ["BCGSI+", "BCGSPIPI+", "BCGSI+1S", "BCGSI+P-2S", "BCGSI+P-1S"]
ctx = bgs.Context(0)


def run(name, n, m, s):
    v = int(bgs.parse_variant(name))
    ld = (n + 31) // 32 * 32
    X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
    Q = torch.empty((m, ld), dtype=torch.float64, device="cuda")
    bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
    try:
        bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        ts = []
        for _ in range(2):
            r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
            ts.append(tm.factor_ms)
        met = bgs.metrics_device(ctx, n, m, n, X.data_ptr(), ld, Q.data_ptr(), ld, r) \
            if hasattr(bgs, "metrics_device") else None
        gf = bgs.variant_flops(v, n, m, s) / (min(ts) * 1e-3) / 1e9
        print(f"{name:11s} n={n:.0e} m={m:4d} s={s:2d}  {min(ts):9.2f} ms  {gf:8.0f} GF/s  {met}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name:11s} n={n:.0e} m={m:4d} s={s:2d}  ERROR {type(e).__name__}: {str(e)[:120]}", flush=True)
    del X, Q
    torch.cuda.empty_cache()


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "s", "s4"):
    for s in ((4,) if which == "s4" else (1, 2, 4, 8, 16)):
        for name in NAMES:
            run(name, 1_000_000, 400, s)
if which in ("all", "shape"):
    for m in (100, 200, 800):
        run("BCGSI+P-1S", 1_000_000, m, 4)
    for n in (100_000, 4_000_000):
        run("BCGSI+P-1S", n, 400, 4)
