"""The reference's command-line driver on the GPU path (paper_2507_21791_b200/cli.py,
blockgs_main.cpp): the key = value sweep-config parser (bench.cpp:136-213) on CPU,
and `bench --config`, `factor`, `verify` end to end on the GPU against the compiled
reference (oracle/_ref) on the same bitwise inputs."""
import io
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_CFGS = "/root/reference/proj/configs"
# same shape as the reference's quick smoke sweep (every variant, two block widths,
# serial and on two simulated processes)
SMALL_CFG = """# quick sweep
n = 64
m = 8
s = 2, 4
kappa = 1e2
procs = 1, 2
seeds = 1
"""


def _cli():
    from paper_2507_21791_b200 import cli
    return cli


def test_parse_small_config_defaults():
    cli = _cli()
    c = cli.parse_bench_config(SMALL_CFG)
    assert c.n_values == [64] and c.m_values == [8] and c.s_values == [2, 4]
    assert c.kappa_values == [100.0] and c.procs_values == [1, 2] and c.seeds == 1
    assert c.variants == [0, 1, 2, 3, 4, 5]  # all_variants() by default
    assert (c.base_seed, c.distribution, c.alpha, c.beta, c.gamma, c.format, c.out) == (
        12345, "geometric", 1e-5, 1e-9, 1e-10, "csv", "")


@pytest.mark.skipif(not os.path.isdir(REF_CFGS), reason="reference configs absent (GPU box)")
def test_parses_every_reference_config():
    cli = _cli()
    for f in sorted(os.listdir(REF_CFGS)):
        if f.endswith(".cfg"):
            c = cli.parse_bench_config_file(os.path.join(REF_CFGS, f))
            assert c.n_values and c.m_values and c.s_values
    c = cli.parse_bench_config_file(os.path.join(REF_CFGS, "stability_sweep.cfg"))
    assert c.variants == [0, 1, 2, 3, 4, 5] and c.kappa_values == [1e1, 1e3, 1e6, 1e10]
    assert c.seeds == 3 and c.distribution == "geometric" and c.format == "csv"
    assert c.out == "stability.csv"


@pytest.mark.parametrize("text,msg", [
    ("n = 64\nm = 8\n", "config: keys n, m, s are required"),
    ("n = 64\nm = 8\ns = 3\n", "config: m = 8 is not a multiple of s = 3"),
    ("n = 4\nm = 8\ns = 4\n", "config: n = 4 is smaller than m = 8"),
    ("n = 64\nm 8\n", "config line 2: expected 'key = value', got 'm 8'"),
    ("n = 64\nsize = 3\n", "config line 2: unknown key 'size'"),
    ("n = 6x4\n", "config line 1: expected an integer, got '6x4'"),
    ("n = 64\nm = 8\ns = 4\nseeds = 1, 2\n", "config line 4: key 'seeds' takes a single value"),
    ("n = 64\nm = 8\ns = 4\nkappa = 0.5\n", "config: kappa must be at least 1"),
    ("n = 64\nm = 8\ns = 4\ndistribution = uniform\n", "unknown distribution 'uniform'"),
    ("n = 64\nm = 8\ns = 4\nformat = xml\n", "config: format must be csv or json"),
    ("n = 64\nm = 8\ns = 4\nvariants = CGS2\n", "unknown variant"),
    ("n =\n", "config line 1: key 'n' has no value"),
])
def test_config_errors_like_reference(text, msg):
    cli = _cli()
    from paper_2507_21791_b200 import api
    with pytest.raises(api.ConfigError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        cli.parse_bench_config(text)


def test_cli_config_error_exit_code(tmp_path):
    p = tmp_path / "bad.cfg"
    p.write_text("n = 64\nm = 8\n")
    r = subprocess.run([sys.executable, "-m", "paper_2507_21791_b200.cli", "bench", "--config",
                        str(p)], cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "error: config: keys n, m, s are required" in r.stderr


def test_gen_matrix_is_the_reference_generator_bitwise(oracle):
    import paper_2507_21791_b200 as bgs
    for (n, m, s, k, seed, g) in [(100, 16, 4, 1e3, 12345, False), (64, 8, 1, 1e2, 7, False),
                                  (333, 24, 3, 1e10, 5, False), (200, 12, 4, 1.0, 9, True)]:
        x = bgs.gen_matrix(n, m, s, k, seed, g)
        y = oracle.gen_matrix(n, m, s, k, seed, g)  # the oracle is pinned to the reference
        assert np.array_equal(x.view(np.int64), y.view(np.int64))


@pytest.mark.gpu
def test_bench_config_end_to_end_matches_reference(tmp_path):
    """The quick-sweep config through `cli bench`: one row per (cell, variant) in the
    reference's column order; counters equal the reference's run on the same X; LOO /
    residual within 10x; predicted_time / speedup from the cost model."""
    from oracle.oracle import Reference
    cfgp = tmp_path / "small.cfg"
    cfgp.write_text(SMALL_CFG + "format = json\n")
    r = subprocess.run([sys.executable, "-m", "paper_2507_21791_b200.cli", "bench", "--config",
                        str(cfgp)], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = json.loads(r.stdout)
    assert len(rows) == 2 * 2 * 6
    import paper_2507_21791_b200 as bgs
    ref = Reference() if Reference.available() else None
    for row in rows:
        assert list(row)[:15] == ["variant", "n", "m", "s", "q", "P", "kappa", "seed_count",
                                  "sync_count", "words_reduced", "flops", "loo", "residual",
                                  "predicted_time", "speedup_vs_bcgsi+"]
        v = int(bgs.parse_variant(row["variant"]))
        assert row["sync_count"] == bgs.expected_syncs(v, row["q"])
        pt = 1e-5 * row["sync_count"] + 1e-9 * row["words_reduced"] + 1e-10 * row["flops"] / row["P"]
        assert row["predicted_time"] == pytest.approx(pt, rel=1e-12)
        assert row["measured_time"] > 0
        if ref is not None:
            x = bgs.gen_matrix(64, 8, 1, 1e2, 12345)
            rr = ref.factor(v, x, row["s"], row["P"], metrics=True)
            assert rr.sync_count == row["sync_count"] and rr.words_reduced == row["words_reduced"]
            assert row["loo"] <= 10 * max(rr.loo, 2.0 ** -53)
            assert row["residual"] <= 10 * max(rr.resid, 2.0 ** -53)


@pytest.mark.gpu
def test_factor_subcommand_csv():
    r = subprocess.run([sys.executable, "-m", "paper_2507_21791_b200.cli", "factor", "--variant",
                        "BCGSI+P-1S", "--n", "1000", "--m", "32", "--s", "4", "--kappa", "1e3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    head, line = r.stdout.strip().splitlines()
    cols = head.split(",")
    vals = dict(zip(cols, line.split(",")))
    assert cols[:15] == ["variant", "n", "m", "s", "q", "P", "kappa", "seed_count", "sync_count",
                         "words_reduced", "flops", "loo", "residual", "predicted_time",
                         "speedup_vs_bcgsi+"]
    assert vals["variant"] == "BCGSI+P-1S" and vals["sync_count"] == "8"
    assert float(vals["loo"]) < 1e-13


@pytest.mark.gpu
def test_verify_subcommand_passes():
    r = subprocess.run([sys.executable, "-m", "paper_2507_21791_b200.cli", "verify"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert sum(l.startswith("PASS ") for l in lines) == 6 and lines[-1] == "all 6 checks passed"
