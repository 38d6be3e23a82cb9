"""Python host mirror of the reference's C++ API for the BCGS QR path, over the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/blockgs/):

* ``VariantId``, ``all_variants``, ``variant_name``, ``parse_variant``,
  ``expected_syncs`` — variant.hpp:8-39 / variant.cpp:17-71
* ``variant_flops`` — cost_model.hpp:37 / cost_model.cpp:29-119
* ``SyncStats`` — sync_stats.hpp:13-27
* ``FactorOutcome`` / ``run_factor`` — runner.hpp:11-29 / runner.cpp:39-67
* ``BcgsOptions`` (probe = RecurrenceProbe) — bcgs.hpp:19-30
* ``gram``, ``tsqr`` — dense_kernels.hpp:15-24, intraorth.hpp:22-27 (building blocks)
* the exception taxonomy — errors.hpp:9-51

All compute goes through ``_lib/libbgs_gpu.so`` (hand-written sm_100a kernels).  There is
no CPU fallback: without a B200 every compute call raises ``CudaError``; without the
built library the import itself fails loudly.
"""
from __future__ import annotations

import ctypes
import enum
import os
import sys
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BGS_LIB_PATH") or os.path.join(_HERE, "_lib", "libbgs_gpu.so")  # override: A/B builds

# ---------------------------------------------------------------------------------------
# errors (errors.hpp:9-51) — codes shared with include/bgs_gpu.h
# ---------------------------------------------------------------------------------------


class Error(RuntimeError):
    """Base class (blockgs::Error)."""


class DimensionError(Error):
    pass


class NotSpdError(Error):
    def __init__(self, msg: str, pivot: int):
        super().__init__(msg)
        self.pivot = pivot


class SingularError(Error):
    def __init__(self, msg: str, index: int):
        super().__init__(msg)
        self.index = index


class RankDeficientError(Error):
    pass


class NonFiniteError(Error):
    pass


class CollectiveError(Error):
    pass


class ConfigError(Error):
    pass


class CudaError(Error):
    """No usable B200 / CUDA failure (the GPU path has no CPU fallback)."""


BGS_OK = 0
_CODE_TO_EXC = {
    1: DimensionError,
    3: SingularError,
    4: RankDeficientError,
    5: NonFiniteError,
    6: CollectiveError,
    7: ConfigError,
    8: Error,
    9: CudaError,
}

# ---------------------------------------------------------------------------------------
# ctypes binding
# ---------------------------------------------------------------------------------------
LABELS_CAP = 65536


class _Stats(ctypes.Structure):
    _fields_ = [
        ("sync_count", ctypes.c_long),
        ("words_reduced", ctypes.c_long),
        ("n_events", ctypes.c_int),
        ("labels", ctypes.c_char * LABELS_CAP),
    ]


class _Err(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int),
        ("pivot", ctypes.c_int),
        ("block", ctypes.c_long),
        ("site", ctypes.c_char * 96),
        ("msg", ctypes.c_char * 1024),
    ]


class _KStat(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 32),
        ("launches", ctypes.c_long),
        ("ms", ctypes.c_double),
        ("alg_bytes", ctypes.c_double),
        ("alg_flops", ctypes.c_double),
    ]


class _Timing(ctypes.Structure):
    _fields_ = [
        ("factor_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("kernel_launches", ctypes.c_long),
    ]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA extension missing: {LIB_PATH} not built. Run `python -c 'import "
            "__graft_entry__ as g; g.build()'` (nvcc, sm_100a). There is no CPU fallback."
        )
    lib = ctypes.CDLL(LIB_PATH)
    P, L, I, D = ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_double
    sig = {
        "bgs_variant_name": ([I], ctypes.c_char_p),
        "bgs_parse_variant": ([ctypes.c_char_p, P, P], I),
        "bgs_expected_syncs": ([I, L], L),
        "bgs_variant_flops": ([I, L, L, L], D),
        "bgs_shard_rows": ([L, I, I, P, P], I),
        "bgs_ctx_create": ([I, I, I, P, P, P], I),
        "bgs_ctx_destroy": ([P], None),
        "bgs_ctx_set_stream": ([P, P], I),
        "bgs_nccl_unique_id": ([P, P], I),
        "bgs_device_info": ([I, P, P, P, L], I),
        "bgs_factor": ([P, I, L, L, L, I, P, L, P, L, P, L, P, P, P], I),
        "bgs_factor_device": ([P, I, L, L, L, L, L, P, L, P, L, P, L, P, P, P], I),
        "bgs_gen_gaussian_device": ([P, ctypes.c_ulonglong, L, L, L, P, L, P], I),
        "bgs_gen_gaussian_host": ([ctypes.c_ulonglong, L, L, P, L], I),
        "bgs_metrics": ([P, L, L, P, L, P, L, P, L, P, P, P], I),
        "bgs_metrics_device": ([P, L, L, L, P, L, P, L, P, L, P, P, P], I),
        "bgs_gram": ([P, P, L, L, P, L, P, P], I),
        "bgs_profile_enable": ([P, I], I),
        "bgs_profile_read": ([P, P, I, P], I),
        "bgs_tsqr": ([P, P, L, L, P, P, P], I),
        "bgs_ctx_create_host_comm": ([I, I, I, P, P, P, P], I),
        "bgs_gen_matrix_host": ([L, L, L, D, ctypes.c_ulonglong, I, P, L, P], I),
        "bgs_factor_opts": ([P, I, L, L, L, I, P, L, P, L, P, L, P, P, P, P], I),
        "bgs_factor_device_opts": ([P, I, L, L, L, L, L, P, L, P, L, P, L, P, P, P, P], I),
        "bgs_ctx_create_peer": ([I, I, I, ctypes.c_ulong, P, P], I),
        "bgs_ctx_peer_handle": ([P, P, P], I),
        "bgs_ctx_peer_attach": ([P, P, I, P], I),
        "bgs_peer_selftest": ([I, I, L, L, I, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = _load()

EXPORTED_SYMBOLS = (
    "bgs_variant_name", "bgs_parse_variant", "bgs_expected_syncs", "bgs_variant_flops",
    "bgs_shard_rows", "bgs_ctx_create", "bgs_ctx_destroy", "bgs_ctx_set_stream",
    "bgs_nccl_unique_id",
    "bgs_device_info", "bgs_factor", "bgs_factor_device", "bgs_gen_gaussian_device",
    "bgs_gen_gaussian_host", "bgs_metrics", "bgs_metrics_device", "bgs_gram", "bgs_tsqr",
    "bgs_profile_enable", "bgs_profile_read", "bgs_ctx_create_host_comm", "bgs_factor_opts",
    "bgs_factor_device_opts", "bgs_gen_matrix_host",
    "bgs_ctx_create_peer", "bgs_ctx_peer_handle", "bgs_ctx_peer_attach", "bgs_peer_selftest",
)

PEER_HANDLE_BYTES = 128

# bgs_allgather_fn / bgs_probe_fn (include/bgs_gpu.h)
_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_ulong)
_PROBE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_long, ctypes.POINTER(ctypes.c_double),
                             ctypes.c_long, ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_double), ctypes.c_long, ctypes.c_int)


class _Options(ctypes.Structure):
    _fields_ = [("classic_intra", ctypes.c_int), ("probe", _PROBE_FN), ("probe_user", ctypes.c_void_p)]


def _raise(rc: int, err: _Err) -> None:
    if rc == BGS_OK:
        return
    msg = err.msg.decode(errors="replace")
    if rc == 2:
        raise NotSpdError(msg, int(err.pivot))
    if rc == 3:
        raise SingularError(msg, int(err.pivot))
    raise _CODE_TO_EXC.get(rc, Error)(msg)


# ---------------------------------------------------------------------------------------
# algorithm-selection API (variant.hpp:8-39)
# ---------------------------------------------------------------------------------------


class VariantId(enum.IntEnum):
    Bcgs = 0  # classic BCGS (classic_impl; BcgsOptions.classic_intra picks TSQR / CholQR)
    BcgsIro = 1  # BCGSI+
    BcgsPipiPlus = 2  # BCGSPIPI+
    BcgsIp1s = 3  # BCGSI+P-1S
    BcgsIp2s = 4  # BCGSI+P-2S
    BcgsI1s = 5  # BCGSI+1S


IN_SCOPE = (VariantId.BcgsIro, VariantId.BcgsPipiPlus, VariantId.BcgsIp1s,
            VariantId.BcgsIp2s, VariantId.BcgsI1s)


def all_variants() -> List[VariantId]:
    return list(VariantId)


def variant_name(v: int) -> str:
    return _lib.bgs_variant_name(int(v)).decode()


def parse_variant(name: str) -> VariantId:
    out = ctypes.c_int()
    err = _Err()
    rc = _lib.bgs_parse_variant(name.encode(), ctypes.byref(out), ctypes.byref(err))
    _raise(rc, err)
    return VariantId(out.value)


def expected_syncs(v: int, q: int) -> int:
    if q < 1:
        raise DimensionError("expected_syncs: q must be at least 1")
    return int(_lib.bgs_expected_syncs(int(v), int(q)))


def variant_flops(v: int, n: int, m: int, s: int) -> float:
    if s < 1 or m < 1 or m % s != 0 or n < m:
        raise DimensionError("variant_flops: need n >= m and m a multiple of s")
    return float(_lib.bgs_variant_flops(int(v), int(n), int(m), int(s)))


def shard_rows(n: int, procs: int, rank: int) -> tuple[int, int]:
    """Ceil row split of distribute() (dist_block.cpp:37-43): (row0, rows)."""
    r0, rows = ctypes.c_long(), ctypes.c_long()
    rc = _lib.bgs_shard_rows(int(n), int(procs), int(rank), ctypes.byref(r0), ctypes.byref(rows))
    if rc:
        raise DimensionError("shard_rows: bad arguments")
    return r0.value, rows.value


# ---------------------------------------------------------------------------------------
# stats / outcome (sync_stats.hpp:13-27, runner.hpp:11-21)
# ---------------------------------------------------------------------------------------


@dataclass
class SyncStats:
    sync_count: int = 0
    words_reduced: int = 0
    label_counts: Dict[str, int] = field(default_factory=dict)
    event_labels: List[str] = field(default_factory=list)

    @classmethod
    def _from(cls, st: _Stats) -> "SyncStats":
        labels = [x for x in st.labels.decode().split("\n") if x] if st.n_events else []
        counts: Dict[str, int] = {}
        for lab in labels:
            counts[lab] = counts.get(lab, 0) + 1
        return cls(int(st.sync_count), int(st.words_reduced), counts, labels)


@dataclass
class Timing:
    factor_ms: float = 0.0
    total_ms: float = 0.0
    kernel_launches: int = 0


@dataclass
class FactorOutcome:
    ok: bool = False
    error: str = ""
    not_spd_pivot: int = 0
    q: Optional[np.ndarray] = None
    r: Optional[np.ndarray] = None
    stats: SyncStats = field(default_factory=SyncStats)
    loo: float = 0.0
    resid: float = 0.0
    x_was_zero: bool = False
    timing: Timing = field(default_factory=Timing)


def peer_selftest(device: int = 0, nranks: int = 4, ng: int = 16, ns: int = 3000,
                  epochs: int = 5) -> None:
    """bgs_peer_selftest: the one-shot exchange protocol with nranks emulated ranks on one
    GPU (pushes, a device synchronize, then the spin flavour of the sum: nothing waits)."""
    err = _Err()
    _raise(_lib.bgs_peer_selftest(int(device), int(nranks), int(ng), int(ns), int(epochs),
                                  ctypes.byref(err)), err)


# ---------------------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------------------


class Context:
    """A device + stream (+ NCCL communicator when nranks > 1, or when an id is given for a
    one-rank context) + workspaces.

    ``host_allgather``: instead of NCCL, a blocking host allgather ``f(bytes) -> bytes``
    (every rank's payload concatenated in rank order), e.g. over torch.distributed gloo
    (``dist.host_allgather``).  Each sync is one call; partials are summed in rank order
    on the host (bgs_ctx_create_host_comm).  Lets several ranks share one GPU.

    ``peer=True``: the one-shot exchange over peer-mapped device windows
    (bgs_ctx_create_peer): after construction every rank passes ``peer_handle()`` of all
    ranks, in rank order, to ``peer_attach`` (``dist.attach_peers`` does both over
    torch.distributed).  No host round trip per sync; NVLink P2P between GPUs, CUDA IPC
    between processes (which may also share one GPU: the wait is then a stream memory
    operation, never a spinning kernel)."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1,
                 nccl_unique_id: Optional[bytes] = None,
                 host_allgather: Optional[Callable[[bytes], bytes]] = None,
                 peer: bool = False, peer_slot_bytes: int = 0):
        self._h = ctypes.c_void_p()
        err = _Err()
        self._cb = None
        if peer:
            rc = _lib.bgs_ctx_create_peer(int(device), int(rank), int(nranks), int(peer_slot_bytes),
                                          ctypes.byref(self._h), ctypes.byref(err))
        elif host_allgather is not None:
            def _ag(user, send, recv, nbytes, _f=host_allgather, _p=int(nranks)):
                try:
                    out = _f(ctypes.string_at(send, nbytes))
                    if len(out) != _p * nbytes:
                        return 1
                    ctypes.memmove(recv, out, len(out))
                    return 0
                except Exception:  # noqa: BLE001  (reported as BGS_E_COLLECTIVE)
                    return 1
            self._cb = _ALLGATHER_FN(_ag)
            rc = _lib.bgs_ctx_create_host_comm(int(device), int(rank), int(nranks),
                                               ctypes.cast(self._cb, ctypes.c_void_p), None,
                                               ctypes.byref(self._h), ctypes.byref(err))
        else:
            uid = None
            if nccl_unique_id is not None:
                uid = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
            rc = _lib.bgs_ctx_create(int(device), int(rank), int(nranks), uid,
                                     ctypes.byref(self._h), ctypes.byref(err))
        _raise(rc, err)
        self.device, self.rank, self.nranks = device, rank, nranks

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def peer_handle(self) -> bytes:
        """This rank's window handle (BGS_PEER_HANDLE_BYTES) for the other ranks."""
        buf = ctypes.create_string_buffer(PEER_HANDLE_BYTES)
        err = _Err()
        _raise(_lib.bgs_ctx_peer_handle(self._h, buf, ctypes.byref(err)), err)
        return buf.raw

    def peer_attach(self, handles, wait_mode: int = 0) -> None:
        """Map every rank's window (handles in rank order).  wait_mode 0: spin in the sum
        kernel when every rank has its own GPU, stream memory operations otherwise."""
        blob = b"".join(bytes(h) for h in handles)
        if len(blob) != PEER_HANDLE_BYTES * self.nranks:
            raise ConfigError("peer_attach needs one handle per rank")
        err = _Err()
        _raise(_lib.bgs_ctx_peer_attach(self._h, ctypes.create_string_buffer(blob, len(blob)),
                                        int(wait_mode), ctypes.byref(err)), err)

    def set_stream(self, stream: int) -> None:
        """cudaStream_t (as an int) whose queued work the *_device calls wait for."""
        _lib.bgs_ctx_set_stream(self._h, ctypes.c_void_p(int(stream) or None))

    def _follow_torch(self) -> None:
        # Device buffers usually come from torch, whose work is queued on its current
        # stream: make the library wait for it (an event; no host synchronisation).
        torch = sys.modules.get("torch")
        if torch is not None and torch.cuda.is_initialized():
            self.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def profile(self, on: bool = True) -> None:
        """Bracket every kernel class of the factorization with CUDA events."""
        _lib.bgs_profile_enable(self._h, 1 if on else 0)

    def read_profile(self) -> Dict[str, Dict[str, float]]:
        """Per kernel class: launches, device ms, algorithmic bytes / flops (resets)."""
        arr = (_KStat * 256)()
        cnt = ctypes.c_int()
        _lib.bgs_profile_read(self._h, arr, 256, ctypes.byref(cnt))
        return {arr[i].name.decode(): dict(launches=int(arr[i].launches), ms=arr[i].ms,
                                           alg_bytes=arr[i].alg_bytes, alg_flops=arr[i].alg_flops)
                for i in range(min(cnt.value, 256))}

    def close(self) -> None:
        if self._h:
            _lib.bgs_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self) -> "Context":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    err = _Err()
    _raise(_lib.bgs_nccl_unique_id(buf, ctypes.byref(err)), err)
    return buf.raw


def _fortran(x: np.ndarray) -> np.ndarray:
    return np.asfortranarray(np.asarray(x, dtype=np.float64))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------------------------------
# run_factor (runner.cpp:39-67)
# ---------------------------------------------------------------------------------------


@dataclass
class BcgsOptions:
    """BcgsOptions (bcgs.hpp:25-30).  ``probe(k, s2, q_local, x_local, shard)`` is
    RecurrenceProbe::on_eval: called once per delayed reprojection of the one-sync variants
    with the 1-based index k of Q_k, the s x s recurrence S2 and this shard's rows of Q_k
    and X_{k+1} (numpy copies)."""
    classic_intra: int = 0
    probe: Optional[Callable[[int, np.ndarray, np.ndarray, np.ndarray, int], None]] = None


def _options(opts: Optional[BcgsOptions]):
    """(ctypes _Options or None, keep-alive) for a call."""
    if opts is None:
        return None, None
    o = _Options()
    o.classic_intra = int(opts.classic_intra)
    cb = None
    if opts.probe is not None:
        def _pr(user, k, s2, s, ql, xl, nl, shard, _f=opts.probe):
            sq = np.ctypeslib.as_array(s2, shape=(s * s,)).reshape((s, s), order="F").copy()
            q = (np.ctypeslib.as_array(ql, shape=(nl * s,)).reshape((nl, s), order="F").copy()
                 if nl else np.zeros((0, s)))
            xx = (np.ctypeslib.as_array(xl, shape=(nl * s,)).reshape((nl, s), order="F").copy()
                  if nl else np.zeros((0, s)))
            _f(int(k), sq, q, xx, int(shard))
        cb = _PROBE_FN(_pr)
        o.probe = cb
    return o, cb


def run_factor(v: int, x: np.ndarray, s: int, procs: int = 1, *, metrics: bool = True,
               ctx: Optional[Context] = None, opts: Optional[BcgsOptions] = None
               ) -> FactorOutcome:
    """Distribute x over `procs` ranks (emulated on one device), factor, gather, measure.

    NotSpd becomes ``ok=False`` with the diagnostic preserved (runner.cpp:56-61); every
    other error raises.  ``metrics`` computes LOO and the relative residual on the GPU.
    """
    ctx = ctx or default_context()
    xf = _fortran(x)
    if xf.ndim != 2:
        raise DimensionError("run_factor: x must be a matrix")
    n, m = xf.shape
    q = np.zeros((n, m), dtype=np.float64, order="F")
    r = np.zeros((m, m), dtype=np.float64, order="F")
    st, tm, err = _Stats(), _Timing(), _Err()
    o, _keep = _options(opts)
    rc = _lib.bgs_factor_opts(ctx.handle, int(v), n, m, int(s), int(procs), _ptr(xf), max(n, 1),
                              _ptr(q), max(n, 1), _ptr(r), max(m, 1),
                              ctypes.byref(o) if o is not None else None, ctypes.byref(st),
                              ctypes.byref(tm), ctypes.byref(err))
    out = FactorOutcome()
    if rc == 2:
        out.ok = False
        out.error = err.msg.decode(errors="replace")
        out.not_spd_pivot = int(err.pivot)
        return out
    _raise(rc, err)
    out.ok = True
    out.q, out.r = q, r
    out.stats = SyncStats._from(st)
    out.timing = Timing(tm.factor_ms, tm.total_ms, int(tm.kernel_launches))
    if metrics:
        out.loo, res = loss_and_residual(xf, q, r, ctx=ctx)
        out.resid = res
        out.x_was_zero = not np.any(xf)
    return out


def loss_and_residual(x: np.ndarray, q: np.ndarray, r: np.ndarray, *,
                      ctx: Optional[Context] = None) -> tuple[float, float]:
    """(||Q^T Q - I||_2, ||X - QR||_F / ||X||_F) on the GPU (metrics.cpp:8-28)."""
    ctx = ctx or default_context()
    xf, qf, rf = _fortran(x), _fortran(q), _fortran(r)
    n, m = xf.shape
    loo, res, err = ctypes.c_double(), ctypes.c_double(), _Err()
    rc = _lib.bgs_metrics(ctx.handle, n, m, _ptr(xf), n, _ptr(qf), n, _ptr(rf), m,
                          ctypes.byref(loo), ctypes.byref(res), ctypes.byref(err))
    _raise(rc, err)
    return loo.value, res.value


def gram(a: np.ndarray, b: np.ndarray, *, ctx: Optional[Context] = None) -> np.ndarray:
    """a^T b through the K1 TMA/DMMA kernel (dense_kernels.hpp:15-24)."""
    ctx = ctx or default_context()
    af, bf = _fortran(a), _fortran(b)
    n, ma = af.shape
    nb, mb = bf.shape
    if nb != n:
        raise DimensionError("gram_accumulate: row counts differ")
    out = np.zeros((ma, mb), dtype=np.float64, order="F")
    err = _Err()
    rc = _lib.bgs_gram(ctx.handle, _ptr(af), n, ma, _ptr(bf), mb, _ptr(out), ctypes.byref(err))
    _raise(rc, err)
    return out


def tsqr(x: np.ndarray, *, ctx: Optional[Context] = None) -> tuple[np.ndarray, np.ndarray]:
    """Economic QR of a tall block through the K4 TSQR kernels (intraorth.hpp:22-27)."""
    ctx = ctx or default_context()
    xf = _fortran(x)
    n, s = xf.shape
    q = np.zeros((n, s), dtype=np.float64, order="F")
    r = np.zeros((s, s), dtype=np.float64, order="F")
    err = _Err()
    rc = _lib.bgs_tsqr(ctx.handle, _ptr(xf), n, s, _ptr(q), _ptr(r), ctypes.byref(err))
    _raise(rc, err)
    return q, r


def gen_matrix(n: int, m: int, s: int = 1, kappa: float = 1.0, seed: int = 0,
               gaussian: bool = False) -> np.ndarray:
    """gen_matrix (matrix_gen.hpp:27, matrix_gen.cpp:18-97), bit for bit: the geometric
    family (default, like MatrixSpec) or the raw Gaussian draws.  Host, one core."""
    x = np.zeros((n, m), dtype=np.float64, order="F")
    err = _Err()
    _raise(_lib.bgs_gen_matrix_host(int(n), int(m), int(s), float(kappa), int(seed),
                                    1 if gaussian else 0, _ptr(x) if x.size else None,
                                    max(int(n), 1), ctypes.byref(err)), err)
    return x


def gen_gaussian_host(seed: int, n: int, m: int) -> np.ndarray:
    """Bitwise port of gen_matrix's Gaussian mode (matrix_gen.cpp:18-56)."""
    x = np.zeros((n, m), dtype=np.float64, order="F")
    rc = _lib.bgs_gen_gaussian_host(int(seed), n, m, _ptr(x), max(n, 1))
    if rc:
        raise DimensionError("gen_gaussian_host: bad shape")
    return x


# ---------------------------------------------------------------------------------------
# device-resident per-rank entry (bcgs.hpp:49-50) — used by bench.py and dist.py
# ---------------------------------------------------------------------------------------


def factor_device(ctx: Context, v: int, n: int, m: int, s: int, row0: int, n_local: int,
                  x_ptr: int, ldx: int, q_ptr: int, ldq: int,
                  opts: Optional[BcgsOptions] = None) -> tuple[np.ndarray, SyncStats, Timing]:
    r = np.zeros((m, m), dtype=np.float64, order="F")
    st, tm, err = _Stats(), _Timing(), _Err()
    ctx._follow_torch()
    o, _keep = _options(opts)
    rc = _lib.bgs_factor_device_opts(ctx.handle, int(v), n, m, s, row0, n_local, x_ptr, ldx,
                                     q_ptr, ldq, _ptr(r), m,
                                     ctypes.byref(o) if o is not None else None,
                                     ctypes.byref(st), ctypes.byref(tm), ctypes.byref(err))
    _raise(rc, err)
    return r, SyncStats._from(st), Timing(tm.factor_ms, tm.total_ms, int(tm.kernel_launches))


def gen_gaussian_device(ctx: Context, seed: int, row0: int, n_local: int, m: int, x_ptr: int,
                        ldx: int) -> None:
    err = _Err()
    ctx._follow_torch()
    rc = _lib.bgs_gen_gaussian_device(ctx.handle, int(seed), row0, n_local, m, x_ptr, ldx,
                                      ctypes.byref(err))
    _raise(rc, err)


def metrics_device(ctx: Context, n: int, m: int, n_local: int, x_ptr: int, ldx: int,
                   q_ptr: int, ldq: int, r: np.ndarray) -> tuple[float, float]:
    rf = _fortran(r)
    loo, res, err = ctypes.c_double(), ctypes.c_double(), _Err()
    ctx._follow_torch()
    rc = _lib.bgs_metrics_device(ctx.handle, n, m, n_local, x_ptr, ldx, q_ptr, ldq, _ptr(rf), m,
                                 ctypes.byref(loo), ctypes.byref(res), ctypes.byref(err))
    _raise(rc, err)
    return loo.value, res.value
