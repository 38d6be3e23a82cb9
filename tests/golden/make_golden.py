"""Generates the committed golden fixtures from the REFERENCE ITSELF (oracle/_ref, the
unmodified reference library compiled from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Outputs (small, committed): tests/golden/factor_golden.npz, tests/golden/gram_lcg.npz.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference  # noqa: E402


def lcg_matrix(rows, cols, seed):
    """The reference tests' LCG fill (tests/oracles.cpp:83-94), restated."""
    mask = (1 << 64) - 1
    state = (seed * 6364136223846793005 + 1442695040888963407) & mask
    m = np.zeros((rows, cols), order="F")
    for j in range(cols):
        for i in range(rows):
            state = (state * 6364136223846793005 + 1442695040888963407) & mask
            m[i, j] = float(state >> 11) * 2.0 ** -52 - 1.0
    return m


CASES = [
    # name, n, m, s, kappa, gaussian, procs
    ("geo_n96_m8_s2_P1", 96, 8, 2, 1e2, False, 1),
    ("geo_n96_m8_s2_P4", 96, 8, 2, 1e2, False, 4),
    ("geo_n200_m16_s4_P3", 200, 16, 4, 1e3, False, 3),
    ("geo_n64_m16_s4_k1e12", 64, 16, 4, 1e12, False, 1),
    ("gau_n150_m12_s3_P2", 150, 12, 3, 1.0, True, 2),
    ("geo_n60_m6_s1_P1", 60, 6, 1, 1e1, False, 1),
    ("geo_n32_m4_s4_P2", 32, 4, 4, 1e2, False, 2),
]


def main():
    ref = Reference()
    arrays = {}
    meta = []
    for name, n, m, s, kappa, gaussian, procs in CASES:
        x = ref.gen_matrix(n, m, s, kappa, 12345, gaussian)
        arrays[f"{name}/x"] = x
        for v in (1, 2, 3, 4, 5):
            res = ref.factor(v, x, s, procs, metrics=True)
            key = f"{name}/v{v}"
            entry = dict(case=name, n=n, m=m, s=s, kappa=kappa, gaussian=gaussian, procs=procs,
                         variant=v, rc=res.rc, sync_count=res.sync_count,
                         words=res.words_reduced, labels=res.labels, pivot=res.pivot,
                         msg=res.msg, loo=res.loo, resid=res.resid)
            if res.rc == 0:
                arrays[f"{key}/q"] = res.q
                arrays[f"{key}/r"] = res.r
            meta.append(entry)
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "factor_golden.npz"), **arrays)

    a = lcg_matrix(40, 7, 77)
    b = lcg_matrix(40, 3, 78)
    np.savez_compressed(os.path.join(HERE, "gram_lcg.npz"), a=a, b=b, g=ref.gram(a, b))
    print("wrote", len(meta), "factorization records")


if __name__ == "__main__":
    main()
