"""Device-side test-matrix generation for the benchmark configurations.

``gen_matrix`` in the reference (matrix_gen.cpp:60-96) builds its geometric test matrices
X = (U diag(sigma)) V^T with U, V the Householder Q factors of seeded Gaussian matrices and
sigma_i = kappa^(-i/(m-1)) — sequentially on one CPU core, which is far too slow for
BASELINE config 5 (n = 1e7, m = 400, kappa = 1e6).  This module builds the same family on
the GPU:

* G (n x m, i.i.d. N(0,1), counter-based Philox: independent of the row sharding) is
  generated with ``bgs_gen_gaussian_device``;
* U = the Q factor of G from this library's own BCGSI+P-1S factorization (R has a
  nonnegative diagonal, so U is the unique QR factor that the reference's sign-fixed
  Householder Q also is — Haar-distributed), row-sharded exactly like X, so a multi-GPU
  run generates its shards in parallel with one NCCL allreduce per block step;
* V (m x m) = Q of a seeded m x m Gaussian (numpy, host; identical on every rank),
  columns sign-fixed to a nonnegative diagonal of R;
* X^T = (V diag(sigma)) U^T — one plain cuBLAS DGEMM (torch.matmul in fp64) per rank.

The bits differ from the reference generator (Philox instead of mt19937_64, BCGS instead
of Householder), the distribution does not.  Parity against the reference runs on the
oracle's own matrices (tests/test_gpu_parity.py feeds gen_matrix's geometric X to the GPU).
"""
from __future__ import annotations

import numpy as np

from . import api


def sigma_schedule(m: int, kappa: float) -> np.ndarray:
    """sigma_i = kappa^(-i/(m-1)) (matrix_gen.cpp:83-90)."""
    if m == 1:
        return np.ones(1)
    return kappa ** (-np.arange(m, dtype=np.float64) / (m - 1))


def haar_orthogonal(m: int, seed: int) -> np.ndarray:
    """Q of a seeded m x m Gaussian with the columns sign-fixed so diag(R) >= 0."""
    g = np.random.default_rng(seed).standard_normal((m, m))
    q, r = np.linalg.qr(g)
    return q * np.where(np.diag(r) < 0.0, -1.0, 1.0)


def geometric_device(ctx: "api.Context", n: int, m: int, kappa: float, seed: int, row0: int,
                     n_local: int, x, ld: int, scratch=None) -> None:
    """Fill x (a torch fp64 CUDA tensor of shape (m, ld): the rank's n_local x m shard,
    column-major) with rows [row0, row0 + n_local) of X = U diag(sigma) V^T.

    `scratch` (same shape as x, optional) holds G; U is written into x first.  On a
    multi-GPU context every rank must call this collectively (the QR of G is distributed).
    """
    import torch

    if scratch is None:
        scratch = torch.empty_like(x)
    api.gen_gaussian_device(ctx, seed, row0, n_local, m, scratch.data_ptr(), ld)
    x.zero_()
    v = int(api.parse_variant("BCGSI+P-1S"))
    s = 4 if m % 4 == 0 else (2 if m % 2 == 0 else 1)
    api.factor_device(ctx, v, n, m, s, row0, n_local, scratch.data_ptr(), ld, x.data_ptr(), ld)
    vs = haar_orthogonal(m, seed ^ 0x5EED) * sigma_schedule(m, kappa)[None, :]
    vs_t = torch.from_numpy(np.ascontiguousarray(vs)).to(device=x.device, dtype=torch.float64)
    # X^T (m x ld) = (V diag(sigma)) @ U^T, U^T being x in its (m, ld) layout
    torch.matmul(vs_t, x, out=scratch)
    x.copy_(scratch)
    if n_local < ld:
        x[:, n_local:].zero_()
