"""Small factorizations for compute-sanitizer (tools/sanitize.sh): every variant, the
fused K12c plans, the merged reduce + step kernel, TSQR, the unfused paths, ragged shards.
Checked against the oracle so a sanitizer run is also a parity run.
    python tools/sanitize_cases.py [quick]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2507_21791_b200 as bgs  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

o = Oracle()
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
cases = [(v, n, m, s, P) for v in (1, 2, 3, 4, 5) for (n, m, s, P) in
         [(300, 24, 4, 1), (333, 36, 3, 2), (700, 32, 8, 1), (260, 32, 16, 1)]]
cases += [(3, 5000, 280, 4, 1), (5, 2000, 64, 4, 3), (0, 300, 24, 4, 1)]
if quick:
    cases = cases[::3]
bad = 0
for (v, n, m, s, P) in cases:
    x = o.gen_matrix(n, m, s, 1e3, 7, False)
    out = bgs.run_factor(v, x, s, P, metrics=True)
    if v == 0:
        ok = out.ok and out.loo < 1e-8
    else:
        ref = o.factor(v, x, s, P, metrics=True)
        ok = out.ok and np.abs(out.r - ref.r).max() <= 1e-10 * np.abs(ref.r).max() and \
            o.loo(out.q) <= 10 * max(ref.loo, 2.0 ** -53)
    bad += not ok
    print(f"v={v} n={n} m={m} s={s} P={P} ok={ok}", flush=True)
print(f"failures: {bad}")
sys.exit(1 if bad else 0)
