"""Host logic of the sweep driver (paper_2507_21791_b200/sweep.py): the reference's report
schema (bench.cpp:383-394), %.17g reals, and the expected-failure rule
(bench.cpp:245-249, variant.cpp:88-104)."""
import io
import math

import pytest


def _sweep():
    try:
        from paper_2507_21791_b200 import sweep
    except ImportError as e:  # the package needs the built library
        pytest.skip(str(e))
    return sweep


def test_schema_and_formatting():
    sweep = _sweep()
    row = {"variant": "BCGSI+P-1S", "n": 100, "m": 8, "s": 4, "q": 2, "P": 1, "kappa": 1.0,
           "seed_count": 1, "sync_count": 2, "words_reduced": 64, "flops": 1.5e4, "loo": 1e-16,
           "residual": 2e-16, "predicted_time": 0.1, "speedup_vs_bcgsi+": 3.0, "gflops": 0.15,
           "hbm_frac": None}
    out = io.StringIO()
    sweep.write([row], "csv", out)
    head, line = out.getvalue().splitlines()
    assert head.split(",")[:15] == ["variant", "n", "m", "s", "q", "P", "kappa", "seed_count",
                                    "sync_count", "words_reduced", "flops", "loo", "residual",
                                    "predicted_time", "speedup_vs_bcgsi+"]
    assert line.split(",")[6] == "1" and line.split(",")[11] == "9.9999999999999998e-17"
    assert sweep.format_real(0.1) == "0.10000000000000001"


def test_expected_failure_rule():
    sweep = _sweep()
    u = 2.0 ** -53
    # P-1S assumes u kappa^2 <= 1: failure expected once u kappa^2 >= 1e-3
    assert not sweep.assumption_violated("BCGSI+P-1S", 1e6)
    assert sweep.assumption_violated("BCGSI+P-1S", math.sqrt(1e-3 / u) * 1.01)
    assert sweep.assumption_violated("BCGSI+1S", 1e5)        # p = 3
    assert not sweep.assumption_violated("BCGSI+", 1e12)     # p = 1: u 1e12 < 1e-3
    assert not sweep.assumption_violated("BCGS", 1e20)       # no usable bound
