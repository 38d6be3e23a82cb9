# NaN-poison sweep (BGS_POISON=1): every variant on ragged / multi-shard / wide shapes against
# the oracle, one fresh context per shape; run under the switches that select other code
# paths (BGS_NO_FUSE, BGS_K12C_PLAN, BGS_NO_MERGE_SMALL, BGS_TSQR_GENERIC, ...).
import sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2507_21791_b200 as bgs
from oracle.oracle import Oracle
o = Oracle()
bad = []
shapes = [(70001, 96, 4, 3), (3000, 800, 4, 1), (20001, 64, 4, 2), (4097, 64, 1, 1), (4097, 64, 2, 3),
          (1500, 48, 6, 2), (6000, 160, 8, 1), (9001, 128, 16, 2), (5003, 36, 4, 1), (7777, 44, 4, 2),
          (3333, 30, 5, 1), (2222, 35, 7, 3), (12345, 52, 4, 1), (999, 60, 12, 2)]
for (n, m, s, P) in shapes:
    x = o.gen_matrix(n, m, s, 1e3, 777, False)
    ctx = bgs.Context(0)
    for v in [1, 2, 3, 4, 5]:
        ref = o.factor(v, x, s, P, metrics=False)
        err = ""
        try:
            out = bgs.run_factor(v, x, s, P, metrics=False, ctx=ctx)
            ok = out.ok and np.abs(out.r - ref.r).max() <= 1e-9 * np.abs(ref.r).max()
            if not out.ok: err = out.error[:60]
            elif not ok: err = "R %.1e" % (np.abs(out.r - ref.r).max() / np.abs(ref.r).max())
        except Exception as e:
            ok = False; err = str(e)[:60]
        if not ok or ref.rc != 0:
            bad.append((v, n, m, s, P, ref.rc, err))
    del ctx
print("ENV", {k: v for k, v in os.environ.items() if k.startswith("BGS_")}, "BAD", bad, flush=True)
