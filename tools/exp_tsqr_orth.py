# Orthogonality of the TSQR Q (leaf kernels A/B): ||Q^T Q - I||_2 and ||X - QR|| / ||X||.
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2507_21791_b200 as bgs
for n, s in [(1_000_000, 4), (100_000, 4), (1024, 4), (4096, 4), (1_000_000, 8), (200_000, 16)]:
    x = bgs.gen_gaussian_host(12345, n, s)
    q, r = bgs.tsqr(x)
    g = q.T @ q - np.eye(s)
    res = np.linalg.norm(x - q @ r) / np.linalg.norm(x)
    # column-wise norms of the leaf blocks (1024 rows)
    print(f"n={n:8d} s={s:2d} loo={np.linalg.norm(g, 2):.3e} res={res:.3e}")
