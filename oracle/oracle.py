"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``Oracle``    : our C restatement (oracle/_build/liboracle.so, oracle/bcgs_oracle.c).
* ``Reference`` : the unmodified reference library compiled from /root/reference by
                  oracle/Makefile (oracle/_ref/libblockgs_ref.so); absent if it was never
                  built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libblockgs_ref.so")

P, L, I, D = ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_double


class _OrStats(ctypes.Structure):
    _fields_ = [("sync_count", L), ("words_reduced", L), ("n_events", I),
                ("labels", ctypes.c_char * 65536), ("pivot", I), ("msg", ctypes.c_char * 1024)]


@dataclass
class Result:
    rc: int
    q: np.ndarray = None
    r: np.ndarray = None
    sync_count: int = 0
    words_reduced: int = 0
    labels: List[str] = field(default_factory=list)
    pivot: int = 0
    msg: str = ""
    seconds: float = 0.0
    loo: float = float("nan")
    resid: float = float("nan")


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        self.lib = ctypes.CDLL(path)
        lib = self.lib
        lib.or_gen_matrix.argtypes = [L, L, L, D, ctypes.c_ulonglong, I, P]
        lib.or_factor.argtypes = [I, P, L, L, L, I, P, P, P]
        lib.or_gram.argtypes = [P, L, L, P, L, P]
        lib.or_householder.argtypes = [P, L, L, P, P]
        lib.or_loo.argtypes = [P, L, L]
        lib.or_loo.restype = D
        lib.or_residual.argtypes = [P, P, P, L, L]
        lib.or_residual.restype = D
        lib.or_variant_flops.argtypes = [I, L, L, L]
        lib.or_variant_flops.restype = D
        lib.or_expected_syncs.argtypes = [I, L]
        lib.or_expected_syncs.restype = L
        lib.or_chol.argtypes = [P, L, P, P]

    def gen_matrix(self, n, m, s, kappa=1e2, seed=12345, gaussian=False):
        x = np.zeros((n, m), order="F")
        rc = self.lib.or_gen_matrix(n, m, s, kappa, seed, 1 if gaussian else 0, x.ctypes.data)
        if rc:
            raise ValueError(f"or_gen_matrix rc={rc}")
        return x

    def factor(self, v, x, s, procs=1, metrics=False) -> Result:
        x = _f(x)
        n, m = x.shape
        q = np.zeros((n, m), order="F")
        r = np.zeros((m, m), order="F")
        st = _OrStats()
        rc = self.lib.or_factor(int(v), x.ctypes.data, n, m, s, procs, q.ctypes.data,
                                r.ctypes.data, ctypes.byref(st))
        res = Result(rc, q, r, st.sync_count, st.words_reduced,
                     [t for t in st.labels.decode().split("\n") if t], st.pivot,
                     st.msg.decode())
        if rc == 0 and metrics:
            res.loo = self.loo(q)
            res.resid = self.residual(x, q, r)
        return res

    def gram(self, a, b):
        a, b = _f(a), _f(b)
        out = np.zeros((a.shape[1], b.shape[1]), order="F")
        self.lib.or_gram(a.ctypes.data, a.shape[0], a.shape[1], b.ctypes.data, b.shape[1],
                         out.ctypes.data)
        return out

    def householder(self, x):
        x = _f(x)
        rows, cols = x.shape
        p = min(rows, cols)
        q = np.zeros((rows, p), order="F")
        r = np.zeros((p, cols), order="F")
        self.lib.or_householder(x.ctypes.data, rows, cols, q.ctypes.data, r.ctypes.data)
        return q, r

    def chol(self, a):
        a = _f(a)
        g = np.zeros_like(a, order="F")
        piv = ctypes.c_int()
        rc = self.lib.or_chol(a.ctypes.data, a.shape[0], g.ctypes.data, ctypes.byref(piv))
        return rc, g, piv.value

    def loo(self, q):
        q = _f(q)
        return self.lib.or_loo(q.ctypes.data, q.shape[0], q.shape[1])

    def residual(self, x, q, r):
        x, q, r = _f(x), _f(q), _f(r)
        return self.lib.or_residual(x.ctypes.data, q.ctypes.data, r.ctypes.data, x.shape[0],
                                    x.shape[1])

    def variant_flops(self, v, n, m, s):
        return self.lib.or_variant_flops(v, n, m, s)

    def expected_syncs(self, v, q):
        return self.lib.or_expected_syncs(v, q)


class Reference:
    """The compiled reference itself (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        self.lib = ctypes.CDLL(path)
        lib = self.lib
        lib.ref_gen_matrix.argtypes = [L, L, L, D, ctypes.c_ulonglong, I, P, P, L]
        lib.ref_factor.argtypes = [I, P, L, L, L, I, I, P, P, P, P, P, L, P, P, P, P, P, L]
        lib.ref_gram.argtypes = [P, L, L, P, L, P]
        lib.ref_householder.argtypes = [P, L, L, P, P]
        lib.ref_loo.argtypes = [P, L, L]
        lib.ref_loo.restype = D
        lib.ref_residual.argtypes = [P, P, P, L, L]
        lib.ref_residual.restype = D
        lib.ref_variant_flops.argtypes = [I, L, L, L]
        lib.ref_variant_flops.restype = D
        lib.ref_expected_syncs.argtypes = [I, L]
        lib.ref_expected_syncs.restype = L
        lib.ref_set_classic_intra.argtypes = [I]
        lib.ref_set_classic_intra.restype = None

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def gen_matrix(self, n, m, s, kappa=1e2, seed=12345, gaussian=False):
        x = np.zeros((n, m), order="F")
        msg = ctypes.create_string_buffer(512)
        rc = self.lib.ref_gen_matrix(n, m, s, kappa, seed, 1 if gaussian else 0, x.ctypes.data,
                                     msg, 512)
        if rc:
            raise ValueError(msg.value.decode())
        return x

    def factor(self, v, x, s, procs=1, metrics=False, want_q=True, classic_intra=0) -> Result:
        self.lib.ref_set_classic_intra(int(classic_intra))
        x = _f(x)
        n, m = x.shape
        q = np.zeros((n, m), order="F") if want_q else None
        r = np.zeros((m, m), order="F")
        sc, w = ctypes.c_long(), ctypes.c_long()
        lab = ctypes.create_string_buffer(65536)
        loo, res, sec = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        piv = ctypes.c_int()
        msg = ctypes.create_string_buffer(1024)
        rc = self.lib.ref_factor(int(v), x.ctypes.data, n, m, s, procs, 1 if metrics else 0,
                                 q.ctypes.data if want_q else None, r.ctypes.data,
                                 ctypes.byref(sc), ctypes.byref(w), lab, 65536,
                                 ctypes.byref(loo), ctypes.byref(res), ctypes.byref(sec),
                                 ctypes.byref(piv), msg, 1024)
        out = Result(rc, q, r, sc.value, w.value,
                     [t for t in lab.value.decode().split("\n") if t], piv.value,
                     msg.value.decode(), sec.value)
        if metrics and rc == 0:
            out.loo, out.resid = loo.value, res.value
        return out

    def variant_flops(self, v, n, m, s):
        """cost_model.cpp:29-119 (the reference's own analytic count)."""
        return self.lib.ref_variant_flops(v, n, m, s)

    def expected_syncs(self, v, q):
        return self.lib.ref_expected_syncs(v, q)

    def gram(self, a, b):
        a, b = _f(a), _f(b)
        out = np.zeros((a.shape[1], b.shape[1]), order="F")
        self.lib.ref_gram(a.ctypes.data, a.shape[0], a.shape[1], b.ctypes.data, b.shape[1],
                          out.ctypes.data)
        return out
