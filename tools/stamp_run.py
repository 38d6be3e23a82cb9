# Debug build only (-DBGS_STEP_STAMPS): globaltimer stamps of the reduce + step kernel and
# the first stage of the next fused kernel, per block step, from one plain factorization.
import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2507_21791_b200 as bgs
from paper_2507_21791_b200 import api
lib = api._lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
m, s = 400, 4
ld = (n + 31) // 32 * 32
ctx = bgs.Context(0)
X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
Q = torch.empty((m, ld), dtype=torch.float64, device="cuda")
bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
st = np.zeros(512 * 8, np.uint64); kt = np.zeros(512 * 8, np.uint64)
for rep in range(2):
    torch.cuda.synchronize()
    lib.bgs_dbg_k12_stamps(ctypes.c_void_p(kt.ctypes.data), 1)
    r, sst, tm = bgs.factor_device(ctx, 3, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
    torch.cuda.synchronize()
lib.bgs_dbg_step_stamps(ctypes.c_void_p(st.ctypes.data))
lib.bgs_dbg_k12_stamps(ctypes.c_void_p(kt.ctypes.data), 0)
st = st.reshape(512, 8).astype(np.int64); kt = kt.reshape(512, 8).astype(np.int64)
print("factor ms", tm.factor_ms)
gaps, rdy, dur, spread, kdur = [], [], [], [], []
for k in range(1, m // s - 1):
    end = st[k, 7]
    e0, e1, w0, w1, x0, x1, r0, r1 = kt[k]
    gaps.append(e0 - end); rdy.append(r1 - end); dur.append(st[k, 7] - st[k, 0])
    spread.append(x1 - x0); kdur.append(x1 - e0)
    if k % 10 == 0:
        print(f"k {k:3d} step {st[k,7]-st[k,0]:6d} ns | vs step end: entry {e0-end:6d}..{e1-end:6d} "
              f"wait released {w0-end:6d}..{w1-end:6d} ready {r0-end:6d}..{r1-end:6d} | "
              f"CTA ends spread {x1-x0:6d} of kernel {x1-e0:7d}")
print("mean step", np.mean(dur), "mean first entry", np.mean(gaps), "mean last ready", np.mean(rdy),
      "mean CTA-end spread", np.mean(spread), "sum spread ms", np.sum(spread) / 1e6)
# per-phase means of the reduce + step kernel: [start, reduce done, detect, pass, products,
# chol, trsm, end] (small.cu STAMP points)
ph = np.diff(st[1:m // s - 1, :8], axis=1).mean(axis=0)
print("phases (ns): reduce %.0f detect %.0f pass %.0f products %.0f chol1 %.0f trsm %.0f chol2+stores %.0f"
      % tuple(ph))
# raw timeline around a few steps (ns, relative to the step kernel's start of step k):
# fused kernel of kp = k s (entry min / ready max / CTA end min, max) and step kernel k
for k in (10, 50, 90):
    if k >= m // s - 1:
        continue
    t0 = st[k, 0]
    e0, e1, w0, w1, x0, x1, r0, r1 = kt[k]
    print(f"k {k}: fused(kp={k * s}) entry {e0 - t0} ready {r1 - t0} end {x0 - t0}..{x1 - t0} | "
          f"step {k}: start 0 reduced {st[k, 1] - t0} end {st[k, 7] - t0} | "
          f"fused(kp={(k + 1) * s}) entry {kt[k + 1, 0] - t0} ready {kt[k + 1, 7] - t0} "
          f"end {kt[k + 1, 4] - t0}..{kt[k + 1, 5] - t0}")
