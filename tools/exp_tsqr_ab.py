# A/B of the TSQR leaf kernels: elementwise Q/R difference and the P-1S factorization LOO.
import os, subprocess, sys, json
sys.path.insert(0, ".")
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2507_21791_b200 as bgs
    x = bgs.gen_gaussian_host(12345, 1_000_000, 4)
    q, r = bgs.tsqr(x)
    np.save(sys.argv[2] + "_q.npy", q); np.save(sys.argv[2] + "_r.npy", r)
    x2 = bgs.gen_gaussian_host(12345, 200_000, 64)
    o = bgs.run_factor(3, x2, 4, 1, metrics=True)
    print(json.dumps({"loo": o.loo, "resid": o.resid}))
    sys.exit(0)
for tag, env in [("reg", {}), ("gen", {"BGS_TSQR_GENERIC": "1"})]:
    out = subprocess.run([sys.executable, __file__, "child", "/tmp/tsqr_" + tag], env={**os.environ, **env},
                         capture_output=True, text=True)
    print(tag, out.stdout.strip(), out.stderr.strip()[-300:])
qa, qb = np.load("/tmp/tsqr_reg_q.npy"), np.load("/tmp/tsqr_gen_q.npy")
ra, rb = np.load("/tmp/tsqr_reg_r.npy"), np.load("/tmp/tsqr_gen_r.npy")
print("max|dQ|", np.abs(qa - qb).max(), "max|dR|/max|R|", np.abs(ra - rb).max() / np.abs(rb).max())
print("colnorm-1 reg", np.linalg.norm(qa, axis=0) - 1, "gen", np.linalg.norm(qb, axis=0) - 1)
