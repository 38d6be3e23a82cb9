# Graph replay with DIFFERENT data than the capturing call: for each (variant, n, m, s) run
# matrix A (plain), matrix B (captures), matrix A (replays) through bgs_factor_device on fixed
# buffers and compare each with a BGS_GRAPH=0 context's result on the same data (bitwise).
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_21791_b200 as bgs
shapes = [(v, n, m, s) for v in (1, 2, 3, 4, 5) for (n, m, s) in [(56, 54, 6), (300, 48, 4), (300, 48, 8), (1000, 30, 3), (20000, 64, 4), (5000, 64, 16)]]
ctx = bgs.Context(0)
bad = 0
for (v, n, m, s) in shapes:
    ld = (n + 31) // 32 * 32
    X = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    mats = [bgs.gen_gaussian_host(11 + i, n, m) for i in range(2)]
    outs = {}
    for mode in ("graph", "plain"):
        if mode == "plain":
            os.environ["BGS_GRAPH"] = "0"
        else:
            os.environ.pop("BGS_GRAPH", None)
        res = []
        for which in (0, 1, 0, 1):
            X.zero_(); Q.zero_()
            X[:, :n] = torch.from_numpy(np.ascontiguousarray(mats[which].T)).cuda()
            try:
                r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
                res.append((r.copy(), Q[:, :n].cpu().numpy().copy()))
            except Exception as e:  # noqa: BLE001
                res.append((np.full((m, m), np.nan), np.full((m, n), np.nan)))
                print("   ", mode, "call", len(res), "EXC", str(e)[:60])
        outs[mode] = res
    ok = all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(outs["graph"], outs["plain"]))
    bad += not ok
    print(("ok  " if ok else "BAD ") + f"v={v} n={n} m={m} s={s}", "" if ok else [float(np.abs(a[0] - b[0]).max()) for a, b in zip(outs["graph"], outs["plain"])])
print("mismatches:", bad)
