# Debug build only (-DBGS_STEP_STAMPS): globaltimer stamps of the reduce + step kernel and
# the first stage of the next fused kernel, per block step, from one plain factorization.
import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2507_21791_b200 as bgs
from paper_2507_21791_b200 import api
lib = api._lib
n, m, s = 1_000_000, 400, 4
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
gaps, rdy, dur = [], [], []
for k in range(1, m // s - 1):
    end = st[k, 7]
    e0, e1, w0, w1, f0, f1, r0, r1 = kt[k] - end
    gaps.append(e0); rdy.append(r1); dur.append(st[k, 7] - st[k, 0])
    if k % 10 == 0:
        print(f"k {k:3d} step {st[k,7]-st[k,0]:6d} ns | relative to step end: entry {e0:6d}..{e1:6d} "
              f"wait released {w0:6d}..{w1:6d} setup done {f0:6d}..{f1:6d} ready {r0:6d}..{r1:6d}")
print("mean step", np.mean(dur), "mean first entry", np.mean(gaps), "mean last ready", np.mean(rdy))
if len(sys.argv) > 1:  # per step: consumer setup time (wait release -> first stage wait), max over CTAs
    print("k setup_ns(min..max)")
    for k in range(1, m // s - 1):
        e0, e1, w0, w1, f0, f1, r0, r1 = kt[k]
        print(k, f0 - w1, f1 - w0)
