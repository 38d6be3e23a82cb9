"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every symbol
include/bgs_gpu.h declares, and its host logic (variant selection, sync formulas, flop
counts, row sharding, the reference generator port) agrees with the oracle.  No compute
calls here: on a host without a GPU the compute entry points must fail loudly."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "bgs_gpu.h")).read()
    return sorted(set(re.findall(r"\b(bgs_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_2507_21791_b200.api as api
    lib = ctypes.CDLL(api.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(api.EXPORTED_SYMBOLS) <= set(syms)


def test_library_is_sm100a_code():
    import subprocess

    import paper_2507_21791_b200.api as api
    out = subprocess.run(["cuobjdump", "--list-elf", api.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_variant_selection_api():
    import paper_2507_21791_b200 as bgs
    names = ["BCGS", "BCGSI+", "BCGSPIPI+", "BCGSI+P-1S", "BCGSI+P-2S", "BCGSI+1S"]
    assert [bgs.variant_name(v) for v in bgs.all_variants()] == names
    for v, nm in enumerate(names):
        assert bgs.parse_variant(nm) == v
        assert bgs.parse_variant(nm.lower()) == v
    with pytest.raises(bgs.api.ConfigError, match="unknown variant"):
        bgs.parse_variant("CGS2")
    with pytest.raises(bgs.api.DimensionError):
        bgs.expected_syncs(3, 0)


def test_sync_formulas_and_flops_match_oracle(oracle):
    import paper_2507_21791_b200 as bgs
    for v in range(6):
        for q in (1, 2, 3, 8, 100):
            assert bgs.expected_syncs(v, q) == oracle.expected_syncs(v, q)
        for (n, m, s) in [(1000, 400, 4), (10**6, 400, 1), (10**7, 400, 16), (100, 10, 5),
                          (64, 64, 64)]:
            assert bgs.variant_flops(v, n, m, s) == oracle.variant_flops(v, n, m, s)


def test_shard_rows_ceil_split():
    import paper_2507_21791_b200 as bgs
    # test_distblock.cpp: 10 rows over P=4 -> 3, 3, 3, 1
    assert [bgs.shard_rows(10, 4, r)[1] for r in range(4)] == [3, 3, 3, 1]
    assert [bgs.shard_rows(10, 4, r)[0] for r in range(4)] == [0, 3, 6, 9]
    # empty trailing ranks (P > n)
    assert [bgs.shard_rows(3, 5, r) for r in range(5)] == [(0, 1), (1, 1), (2, 1), (3, 0), (3, 0)]


def test_host_generator_is_bitwise_reference(oracle):
    import paper_2507_21791_b200 as bgs
    for (n, m, seed) in [(1, 1, 0), (97, 5, 12345), (1000, 8, 2024)]:
        a = bgs.gen_gaussian_host(seed, n, m)
        b = oracle.gen_matrix(n, m, 1, 1.0, seed, True)
        assert np.array_equal(a.view(np.int64), b.view(np.int64))


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2507_21791_b200 as bgs
    with pytest.raises(bgs.api.CudaError, match="no CPU fallback"):
        bgs.Context(0)
