"""Pins the CPU oracle (oracle/bcgs_oracle.c) before any GPU result is judged by it.

* bitwise against golden fixtures produced by the REFERENCE ITSELF
  (tests/golden/make_golden.py over oracle/_ref): Q, R, sync counts, word counts, event
  labels, NotSpd pivot + message, exact LOO and residual;
* bitwise against the live reference library when oracle/_ref is present;
* the exact Gram against rational arithmetic (correct rounding, dense_kernels.hpp:18);
* known answers of the reference's own unit tests (test_dense_core.cpp,
  test_intraorth.cpp, test_bcgs.cpp, test_distblock.cpp).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def bits(a):
    return np.ascontiguousarray(a).view(np.int64)


@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(GOLD, "factor_golden.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def test_oracle_bitwise_matches_reference_goldens(oracle, golden):
    z, meta = golden
    checked = 0
    for e in meta:
        x = z[f"{e['case']}/x"]
        res = oracle.factor(e["variant"], x, e["s"], e["procs"], metrics=e["rc"] == 0)
        assert res.rc == e["rc"], e
        if e["rc"] != 0:
            assert res.pivot == e["pivot"] and res.msg == e["msg"]
            continue
        key = f"{e['case']}/v{e['variant']}"
        assert np.array_equal(bits(res.q), bits(z[key + "/q"])), key
        assert np.array_equal(bits(res.r), bits(z[key + "/r"])), key
        assert res.sync_count == e["sync_count"] and res.words_reduced == e["words"]
        assert res.labels == e["labels"]
        assert res.loo == e["loo"] and res.resid == e["resid"]
        checked += 1
    assert checked >= 30


def test_oracle_generator_matches_reference_goldens(oracle, golden):
    z, meta = golden
    seen = set()
    for e in meta:
        if e["case"] in seen:
            continue
        seen.add(e["case"])
        x = oracle.gen_matrix(e["n"], e["m"], e["s"], e["kappa"], 12345, e["gaussian"])
        assert np.array_equal(bits(x), bits(z[f"{e['case']}/x"])), e["case"]


def test_oracle_matches_live_reference(oracle):
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built on this host")
    ref = Reference()
    for (n, m, s, kappa, gauss, procs) in [(120, 12, 3, 1e4, False, 5), (500, 20, 4, 1.0, True, 2),
                                           (1000, 32, 8, 1e6, False, 3)]:
        x = ref.gen_matrix(n, m, s, kappa, 2024, gauss)
        assert np.array_equal(bits(x), bits(oracle.gen_matrix(n, m, s, kappa, 2024, gauss)))
        for v in (1, 2, 3, 4, 5):
            a = ref.factor(v, x, s, procs)
            b = oracle.factor(v, x, s, procs)
            assert a.rc == b.rc
            if a.rc:
                assert a.msg == b.msg and a.pivot == b.pivot
                continue
            assert np.array_equal(bits(a.q), bits(b.q)) and np.array_equal(bits(a.r), bits(b.r))
            assert (a.sync_count, a.words_reduced, a.labels) == (b.sync_count, b.words_reduced,
                                                               b.labels)


def _exact_gram(a, b):
    out = np.zeros((a.shape[1], b.shape[1]))
    for i in range(a.shape[1]):
        for j in range(b.shape[1]):
            acc = Fraction(0)
            for k in range(a.shape[0]):
                acc += Fraction(float(a[k, i])) * Fraction(float(b[k, j]))
            out[i, j] = float(acc)  # Fraction -> float rounds to nearest-even
    return out


def test_exact_gram_is_correctly_rounded(oracle):
    z = np.load(os.path.join(GOLD, "gram_lcg.npz"))
    g = oracle.gram(z["a"], z["b"])
    assert np.array_equal(bits(g), bits(z["g"]))
    assert np.array_equal(bits(g), bits(_exact_gram(z["a"], z["b"])))
    # catastrophic cancellation is resolved exactly
    a = np.array([[1e16], [1.0], [-1e16]])
    b = np.array([[1.0], [1.0], [1.0]])
    assert oracle.gram(a, b)[0, 0] == 1.0


def test_dense_known_answers(oracle):
    # gram of the worked example (test_dense_core.cpp:78-83)
    x = np.array([[1.0], [2.0], [2.0]])
    assert oracle.gram(x, x)[0, 0] == 9.0
    # cholesky of [[4,2],[2,3]] and the 1-based failing pivot (test_dense_core.cpp:104-131)
    rc, g, _ = oracle.chol(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert rc == 0 and g[0, 0] == 2.0 and g[0, 1] == 1.0 and g[1, 0] == 0.0
    rc, _, piv = oracle.chol(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert rc == 2 and piv == 2
    rc, _, piv = oracle.chol(np.array([[-1.0]]))
    assert rc == 2 and piv == 1
    # householder of the 3-4-5 column (test_dense_core.cpp:168-174)
    q, r = oracle.householder(np.array([[3.0], [4.0]]))
    assert r[0, 0] == 5.0 and abs(q[0, 0] - 0.6) <= 1e-15 and abs(q[1, 0] - 0.8) <= 1e-15


def test_sync_formulas_and_flops(oracle):
    # expected_syncs table (test_bcgs.cpp:61-70)
    assert [oracle.expected_syncs(v, 8) for v in range(6)] == [15, 29, 15, 8, 15, 8]
    assert all(oracle.expected_syncs(v, 1) == 1 for v in range(6))
    # variant_flops of P-1S at config 2
    assert oracle.variant_flops(3, 1000000, 400, 4) == pytest.approx(6.463e11, rel=1e-3)


@pytest.mark.parametrize("q", [2, 4, 8, 16])
def test_oracle_sync_counts(oracle, q):
    x = oracle.gen_matrix(64, 32, 2, 1e1)[:, : q * 2]
    for v in (1, 2, 3, 4, 5):
        for procs in (1, 3):
            res = oracle.factor(v, x, 2, procs)
            assert res.rc == 0 and res.sync_count == oracle.expected_syncs(v, q)
