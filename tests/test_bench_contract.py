"""bench.py keeps the driver's JSON contract: one line on stdout with the contract keys,
for the reference arm (CPU, runs here) and for this library's arm (one B200, small shape)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[-2000:]  # exactly one JSON line
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1")
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GFLOP/s"
    assert d["config"]["workload"].startswith("BCGSI+P-1S n=1000000 m=400 s=4")
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_nonzero_rank_is_silent():
    """Under torchrun (N > 1) only rank 0 runs the reference arm; other ranks exit 0
    without output or work."""
    env = dict(os.environ, RANK="1", LOCAL_RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                        "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = run_bench("--n", "200000", "--m", "64", "--steps", "2", "--warmup", "3",
                  "--cpu-seconds", "1")
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["higher_is_better"] is True
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * 200000 * 64
    assert e["d2h_bytes_per_step"] >= 8 * 200000 * 64
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and 0 < rf["frac"] <= 1.0 and rf["peak"] > 0
    assert d["gpu_launches"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    v = d["verify"]
    assert v["sync_count"] == v["expected_syncs"] == 16 and v["loo"] < 1e-14


def test_reference_arm_loads_nothing_of_the_product():
    """The reference arm runs the reference's own code only: the product package is not
    imported and libbgs_gpu.so is not mapped; ms_per_step is the measured sample time."""
    code = (
        "import sys, json, io, contextlib; sys.argv=['bench.py','--impl','reference','--steps','1',"
        "'--warmup','0','--cpu-seconds','1']; import bench; buf=io.StringIO()\n"
        "with contextlib.redirect_stdout(buf): bench.main()\n"
        "maps=open('/proc/self/maps').read(); d=json.loads(buf.getvalue())\n"
        "print(json.dumps({'pkg': any(m.startswith('paper_2507_21791_b200') for m in sys.modules),"
        "'lib': 'libbgs_gpu' in maps, 'ref': 'libblockgs_ref' in maps or 'liboracle' in maps,"
        "'line': d}))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert not out["pkg"] and not out["lib"] and out["ref"]
    d = out["line"]
    rows = d["sample_rows"]
    assert 400 <= rows <= 1_000_000 and str(rows) in d["cpu_baseline"]["sample"]
    assert "note" not in d  # nothing extrapolated
    assert d["steps"] == 1
