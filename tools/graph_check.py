import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_21791_b200 as bgs
for n, m, s in [(125000, 400, 4), (1000000, 400, 4), (100000, 64, 4), (20000, 64, 8)]:
    ctx = bgs.Context(0)
    ld = (n + 31) // 32 * 32
    X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
    Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
    res = {}
    for mode in ("0", "1"):
        os.environ["BGS_GRAPH"] = mode
        ts, rs = [], []
        for _ in range(8):
            r, st, tm = bgs.factor_device(ctx, 3, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
            ts.append(tm.factor_ms); rs.append(r.copy())
        res[mode] = (np.median(ts[3:]), rs[-1], st.sync_count, list(st.event_labels), tm.kernel_launches, tm.total_ms)
    same = np.array_equal(res["0"][1], res["1"][1]) and res["0"][2:4] == res["1"][2:4]
    print(f"n={n} m={m} s={s}: stream {res['0'][0]:.3f} ms (host {res['0'][5]:.2f}) | graph {res['1'][0]:.3f} ms (host {res['1'][5]:.2f}) | bitwise same R and stats: {same}, launches {res['0'][4]} / {res['1'][4]}")
