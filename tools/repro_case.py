# Re-run one fuzzer case under several code paths: python tools/repro_case.py v n m s P kappa gauss seed
import os, subprocess, sys
args = sys.argv[1:9]
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2507_21791_b200 as bgs
from oracle.oracle import Oracle
v, n, m, s, P = (int(a) for a in sys.argv[1:6]); kappa = float(sys.argv[6]); gauss = sys.argv[7] == "True"; seed = int(sys.argv[8])
o = Oracle()
x = o.gen_matrix(n, m, s, kappa, seed, gauss)
ref = o.factor(v, x, s, P, metrics=True)
env = [o.factor(v, x, s, p, metrics=True).loo for p in (1, 2, 3, 4)]
out = bgs.run_factor(v, x, s, P, metrics=False)
print("oracle loo %.2e (P=1..4: %s) cond %.2e | gpu loo %.2e ratio %.1f dR %.1e" % (ref.loo, " ".join("%.1e" % e for e in env),
      np.linalg.cond(x), o.loo(out.q), o.loo(out.q) / max(ref.loo, 2.0**-53), np.abs(out.r - ref.r).max() / np.abs(ref.r).max()))
'''
for name, env in [("default", {}), ("BGS_K2M=0", {"BGS_K2M": "0"}), ("BGS_NO_FUSE=1", {"BGS_NO_FUSE": "1"}),
                  ("BGS_COMP_TAIL=0", {"BGS_COMP_TAIL": "0"}), ("BGS_COMP_TAIL=all", {"BGS_COMP_TAIL": "all"})]:
    out = subprocess.run([sys.executable, "-c", code] + args, env=dict(os.environ, **env), capture_output=True, text=True)
    print(f"{name:18s}", out.stdout.strip() or out.stderr.strip()[-300:])
