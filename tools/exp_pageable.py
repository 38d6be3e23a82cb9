# bgs_factor (the run_factor drop-in) from pageable vs pinned host buffers at config 2, and
# the cost of pinning the caller's buffers in place (cudaHostRegister).
import ctypes, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_21791_b200 as bgs
from paper_2507_21791_b200 import api
n, m, s = 1_000_000, 400, 4
ctx = bgs.default_context()
x = np.asfortranarray(np.random.default_rng(1).standard_normal((n, m)))
q = np.zeros((n, m), order="F"); q[:] = 0.0  # touch the pages
r = np.zeros((m, m), order="F")
def call():
    st, tm, err = api._Stats(), api._Timing(), api._Err()
    t0 = time.perf_counter()
    rc = api._lib.bgs_factor(ctx.handle, 3, n, m, s, 1, api._ptr(x), n, api._ptr(q), n, api._ptr(r), m,
                             ctypes.byref(st), ctypes.byref(tm), ctypes.byref(err))
    assert rc == 0, err.msg
    return (time.perf_counter() - t0) * 1e3, tm.total_ms
for _ in range(2): print("pageable", call())
cr = torch.cuda.cudart()
t0 = time.perf_counter()
assert cr.cudaHostRegister(x.ctypes.data, x.nbytes, 0) == 0
assert cr.cudaHostRegister(q.ctypes.data, q.nbytes, 0) == 0
print("register 6.4 GB ms", (time.perf_counter() - t0) * 1e3)
for _ in range(2): print("registered", call())
t0 = time.perf_counter()
cr.cudaHostUnregister(x.ctypes.data); cr.cudaHostUnregister(q.ctypes.data)
print("unregister ms", (time.perf_counter() - t0) * 1e3)
