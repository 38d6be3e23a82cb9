# One-off parity check at the headline shape (BASELINE config 2: BCGSI+P-1S, n=1e6, m=400,
# s=4, i.i.d. N(0,1), seed 12345): the UNMODIFIED reference (oracle/_ref, all host threads)
# and this library on the same X bits; R compared entrywise, LOO and residual of both Q
# measured with the same device metrics (double-double).  Writes gpurun_out/config2_parity.json
# and the golden fixture gpurun_out/config2_ref.npz (-> tests/golden/, test_gpu_config2.py).
#   python tools/config2_parity.py      (one B200 box; ~6 min, mostly the reference)
import json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2507_21791_b200 as bgs
from oracle.oracle import Reference

n, m, s, v = 1_000_000, 400, 4, 3
procs = os.cpu_count() or 1
ref = Reference()
t0 = time.time()
x = ref.gen_matrix(n, m, s, 1.0, 12345, True)
t_gen = time.time() - t0
t0 = time.time()
rr = ref.factor(v, x, s, procs, metrics=False, want_q=True)
t_ref = time.time() - t0
assert rr.rc == 0, rr.msg
out = bgs.run_factor(v, x, s, 1, metrics=False)
assert out.ok, out.error
mx = np.max(np.abs(rr.r))
dr = np.abs(out.r - rr.r)
big = np.abs(rr.r) >= 1e-3 * mx
loo_g, res_g = bgs.api.loss_and_residual(x, out.q, out.r)
loo_r, res_r = bgs.api.loss_and_residual(x, rr.q, rr.r)
rep = {
    "workload": "BCGSI+P-1S n=1000000 m=400 s=4 fp64 i.i.d. N(0,1) seed 12345 (BASELINE config 2)",
    "reference": f"oracle/_ref (unmodified reference sources) run_factor, P={procs} host threads, {t_ref:.1f} s",
    "gpu": f"libbgs_gpu bgs_factor (run_factor drop-in), one B200, {out.timing.total_ms:.1f} ms end to end",
    "R_max_abs_diff_over_max_abs": float(np.max(dr) / mx),
    "R_max_entrywise_rel_diff_big": float(np.max(dr[big] / np.abs(rr.r)[big])),
    "R_tolerance": 1e-10,
    "loo": {"gpu": loo_g, "reference": loo_r, "ratio": loo_g / loo_r},
    "residual": {"gpu": res_g, "reference": res_r, "ratio": res_g / res_r},
    "sync_count": {"gpu": out.stats.sync_count, "reference": rr.sync_count},
    "words_reduced": {"gpu": out.stats.words_reduced, "reference": rr.words_reduced},
    "labels_equal": out.stats.event_labels == rr.labels,
    "lower_triangle_exact_zero": bool(np.all(np.tril(out.r, -1) == 0.0)),
    "diag_nonnegative": bool(np.all(np.diag(out.r) >= 0.0)),
    "metrics": "LOO = ||I - Q^T Q||_2 and ||X - QR||_F / ||X||_F for both Q by the same device kernels",
    "gen_seconds": t_gen,
}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rep, open("gpurun_out/config2_parity.json", "w"), indent=1)
# golden fixture for tests/test_gpu_config2.py: the reference's R and accounting at config 2
np.savez_compressed("gpurun_out/config2_ref.npz", r=rr.r, loo=loo_r, resid=res_r,
                    sync_count=rr.sync_count, words=rr.words_reduced,
                    labels=np.array(rr.labels), seconds=t_ref, procs=procs)
print(json.dumps(rep, indent=1))
