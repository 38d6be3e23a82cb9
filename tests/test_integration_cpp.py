"""The reference-side C++ binding (integration/runner_gpu.cpp): blockgs::gpu::run_factor,
compiled against the reference's own headers, compared with the reference's run_factor
(oracle/_ref) by integration/_build/test_runner_gpu: R to 1e-10, LOO / residual within
10x, identical SyncStats, acceptance C8 through BcgsOptions::probe, the error contract."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_runner_gpu")


def test_binding_is_built_and_links_the_c_abi():
    assert os.path.exists(BIN), "run __graft_entry__.build() (make -C integration)"
    syms = subprocess.run(["nm", "-C", BIN], capture_output=True, text=True).stdout
    assert "blockgs::gpu::run_factor" in syms
    assert "bgs_factor_opts" in syms  # the C ABI entry it binds (undefined: from libbgs_gpu.so)
    libs = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libbgs_gpu.so" in libs and "libblockgs_ref.so" in libs and "not found" not in libs


@pytest.mark.gpu
def test_cpp_binding_matches_reference_run_factor():
    r = subprocess.run([BIN], cwd=ROOT, capture_output=True, text=True, timeout=900)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    bad = [l for l in lines if l.get("pass") is False]
    assert r.returncode == 0 and not bad, (r.stdout[-4000:], r.stderr[-2000:])
    checks = [l.get("check") for l in lines]
    assert checks.count("factor") == 7 and checks.count("C8") == 2
    assert {"not_spd", "dimension_error", "non_finite"} <= set(checks)
    assert lines[-1] == {"summary": True, "failures": 0}
