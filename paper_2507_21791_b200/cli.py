"""The reference's command-line driver (proj/tools/blockgs_main.cpp) on the GPU path.

    python -m paper_2507_21791_b200.cli bench  --config F [--cost-alpha A --cost-beta B --cost-gamma G]
    python -m paper_2507_21791_b200.cli factor --variant V --n N --m M --s S [--kappa K]
                                               [--seed X] [--procs P] [--out csv|json]
                                               [--distribution geometric|gaussian]
    python -m paper_2507_21791_b200.cli verify

* ``bench`` reads the reference's ``key = value`` sweep configs (proj/configs/*.cfg) with
  the same keys, defaults, list syntax, comments and ConfigError wording
  (parse_bench_config, bench.cpp:136-213; validate_config, :93-131) and runs run_bench's
  sweep (bench.cpp:253-375): matrices from gen_matrix(n, m, s=1, kappa, seed) -- bit for
  bit, bgs_gen_matrix_host --, the BCGSI+ s = 1 baseline per cell, seeds averaged, NotSpd
  cells as failed rows flagged expected / unexpected.  Each factorization runs on the GPU
  (run_factor through the C ABI, `procs` ranks emulated on the device).  The report is the
  reference's CSV / JSON (write_csv / write_json, bench.cpp:383-420) column for column:
  predicted_time and speedup_vs_bcgsi+ from the config's alpha-beta-gamma cost model
  (cost_model.cpp:7-27) exactly as the reference computes them; two columns are appended,
  measured_time (device seconds of the factorization, mean over seeds) and gflops.
* ``factor`` is run_factor_command (blockgs_main.cpp:62-92): a one-cell sweep.
* ``verify`` is the built-in invariant suite (verify_suite.cpp:43-194) run against the GPU
  path; PASS / FAIL per check, exit 0 iff all pass.  One check is restated: the reference
  demands bitwise-identical Q and R across process counts (its exact Gram makes them
  so); the GPU Gram is fp64 with fixed-order double-double reductions, so across P the
  results agree to rounding (1e-13 relative), not bitwise -- the check says so.

Exit codes as blockgs_main.cpp:131-145: 0 ok, 1 failure (an unexpected abort, a failed
check, any error), 2 ConfigError.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import api

U_ROUND = 2.0 ** -53
EXPECTED_FAILURE_LEVEL = 1e-3  # bench.cpp:24-27
# loo_assumption(v).kappa_power (variant.cpp:88-104)
KAPPA_POWER = {"BCGS": 0, "BCGSI+": 1, "BCGSPIPI+": 2, "BCGSI+P-1S": 2, "BCGSI+P-2S": 1,
               "BCGSI+1S": 3}
COLUMNS = ["variant", "n", "m", "s", "q", "P", "kappa", "seed_count", "sync_count",
           "words_reduced", "flops", "loo", "residual", "predicted_time", "speedup_vs_bcgsi+"]
EXTRA = ["measured_time", "gflops"]


class ConfigError(api.ConfigError):
    pass


# ---------------------------------------------------------------------------------------
# config (bench.hpp:17-33, bench.cpp:29-213)
# ---------------------------------------------------------------------------------------
@dataclass
class BenchConfig:
    variants: List[int] = field(default_factory=lambda: [int(v) for v in api.all_variants()])
    n_values: List[int] = field(default_factory=list)
    m_values: List[int] = field(default_factory=list)
    s_values: List[int] = field(default_factory=list)
    kappa_values: List[float] = field(default_factory=lambda: [1e2])
    procs_values: List[int] = field(default_factory=lambda: [1])
    seeds: int = 3
    base_seed: int = 12345
    distribution: str = "geometric"
    alpha: float = 1e-5
    beta: float = 1e-9
    gamma: float = 1e-10
    out: str = ""
    format: str = "csv"


def _parse_long(item: str, line_no: int) -> int:
    try:
        if item.strip() != item or not item:
            raise ValueError(item)
        return int(item, 10)
    except ValueError:
        raise ConfigError(f"config line {line_no}: expected an integer, got '{item}'") from None


def _parse_double(item: str, line_no: int) -> float:
    try:
        return float(item)
    except ValueError:
        raise ConfigError(f"config line {line_no}: expected a number, got '{item}'") from None


def _distribution(name: str, line_no: int) -> str:
    if name in ("geometric", "geometric-singular-values"):
        return "geometric"
    if name in ("gaussian", "random-gaussian"):
        return "gaussian"
    raise ConfigError(f"config line {line_no}: unknown distribution '{name}' "
                      "(expected geometric or gaussian)")


def validate_config(c: BenchConfig) -> None:
    """validate_config (bench.cpp:93-131)."""
    if not c.n_values or not c.m_values or not c.s_values:
        raise ConfigError("config: keys n, m, s are required")
    if not c.variants:
        raise ConfigError("config: variant list is empty")
    if c.seeds < 1:
        raise ConfigError("config: seeds must be at least 1")
    if c.format not in ("csv", "json"):
        raise ConfigError("config: format must be csv or json")
    if c.alpha < 0 or c.beta < 0 or c.gamma < 0:
        raise ConfigError("config: alpha, beta, gamma must be nonnegative")
    if any(n < 1 for n in c.n_values):
        raise ConfigError("config: n must be positive")
    if any(m < 1 for m in c.m_values):
        raise ConfigError("config: m must be positive")
    if any(s < 1 for s in c.s_values):
        raise ConfigError("config: s must be positive")
    if any(not (k >= 1.0) for k in c.kappa_values):
        raise ConfigError("config: kappa must be at least 1")
    if any(p < 1 for p in c.procs_values):
        raise ConfigError("config: procs must be at least 1")
    for m in c.m_values:
        for s in c.s_values:
            if m % s:
                raise ConfigError(f"config: m = {m} is not a multiple of s = {s}")
        for n in c.n_values:
            if n < m:
                raise ConfigError(f"config: n = {n} is smaller than m = {m}")


def parse_bench_config(text: str) -> BenchConfig:
    """parse_bench_config (bench.cpp:136-204): '#' comments anywhere, 'key = value',
    comma-separated sweep lists, single-valued keys checked."""
    c = BenchConfig()
    for line_no, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip(" \t\r")
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"config line {line_no}: expected 'key = value', got '{line}'")
        key, value = (t.strip(" \t\r") for t in line.split("=", 1))
        items = [t.strip(" \t\r") for t in value.split(",") if t.strip(" \t\r")]
        if not items:
            raise ConfigError(f"config line {line_no}: key '{key}' has no value")

        def single():
            if len(items) != 1:
                raise ConfigError(f"config line {line_no}: key '{key}' takes a single value, "
                                  "not a sweep list")
            return items[0]

        if key == "variants":
            c.variants = [int(api.parse_variant(t)) for t in items]
        elif key == "n":
            c.n_values = [_parse_long(t, line_no) for t in items]
        elif key == "m":
            c.m_values = [_parse_long(t, line_no) for t in items]
        elif key == "s":
            c.s_values = [_parse_long(t, line_no) for t in items]
        elif key == "kappa":
            c.kappa_values = [_parse_double(t, line_no) for t in items]
        elif key == "procs":
            c.procs_values = [_parse_long(t, line_no) for t in items]
        elif key == "seeds":
            c.seeds = _parse_long(single(), line_no)
        elif key == "seed":
            c.base_seed = _parse_long(single(), line_no)
        elif key == "distribution":
            c.distribution = _distribution(single(), line_no)
        elif key in ("alpha", "beta", "gamma"):
            setattr(c, key, _parse_double(single(), line_no))
        elif key == "out":
            c.out = single()
        elif key == "format":
            c.format = single()
        else:
            raise ConfigError(f"config line {line_no}: unknown key '{key}'")
    validate_config(c)
    return c


def parse_bench_config_file(path: str) -> BenchConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(f"cannot open config file '{path}'") from None
    return parse_bench_config(text)


# ---------------------------------------------------------------------------------------
# cost model (cost_model.cpp:7-27) and the sweep (bench.cpp:253-375)
# ---------------------------------------------------------------------------------------
def predicted_time(alpha, beta, gamma, procs, syncs, words, flops) -> float:
    if alpha < 0 or beta < 0 or gamma < 0:
        raise ConfigError("cost model: alpha, beta, gamma must be nonnegative")
    if procs < 1:
        raise ConfigError("cost model: process count must be at least 1")
    return alpha * syncs + beta * words + gamma * flops / procs


def assumption_violated(name: str, kappa: float) -> bool:
    p = KAPPA_POWER.get(name, 0)
    return p > 0 and U_ROUND * kappa ** p >= EXPECTED_FAILURE_LEVEL


def format_real(v: float) -> str:
    return "%.17g" % v


@dataclass
class BenchReport:
    rows: List[dict] = field(default_factory=list)
    exit_code: int = 0


def run_bench(cfg: BenchConfig, ctx: Optional[api.Context] = None, log=sys.stderr) -> BenchReport:
    validate_config(cfg)
    ctx = ctx or api.default_context()
    rep = BenchReport()
    mats: Dict[Tuple, np.ndarray] = {}
    base: Dict[Tuple, Tuple[int, int, float]] = {}

    def matrix_for(n, m, kappa, seed):
        k = (n, m, kappa, seed)
        if k not in mats:  # spec.s = 1 (bench.cpp:262-266)
            mats[k] = api.gen_matrix(n, m, 1, kappa, seed, cfg.distribution == "gaussian")
        return mats[k]

    def baseline_for(n, m, kappa, procs):
        k = (n, m, kappa, procs)
        if k not in base:
            x = matrix_for(n, m, kappa, cfg.base_seed)
            b = api.run_factor(int(api.VariantId.BcgsIro), x, 1, procs, metrics=False, ctx=ctx)
            if not b.ok:
                raise api.Error("bench: the BCGSI+ baseline run aborted unexpectedly: " + b.error)
            base[k] = (b.stats.sync_count, b.stats.words_reduced,
                       api.variant_flops(int(api.VariantId.BcgsIro), n, m, 1))
        return base[k]

    for n in cfg.n_values:
        for m in cfg.m_values:
            for s in cfg.s_values:
                for kappa in cfg.kappa_values:
                    for procs in cfg.procs_values:
                        b = baseline_for(n, m, kappa, procs)
                        t_base = predicted_time(cfg.alpha, cfg.beta, cfg.gamma, procs, *b)
                        for v in cfg.variants:
                            name = api.variant_name(v)
                            row = {"variant": name, "n": n, "m": m, "s": s, "q": m // s,
                                   "P": procs, "kappa": kappa, "seed_count": cfg.seeds,
                                   "sync_count": 0, "words_reduced": 0,
                                   "flops": api.variant_flops(v, n, m, s)}
                            loos, ress, times = [], [], []
                            failed, err, counters = False, "", None
                            for i in range(cfg.seeds):
                                x = matrix_for(n, m, kappa, cfg.base_seed + i)
                                run = api.run_factor(v, x, s, procs, metrics=True, ctx=ctx)
                                if not run.ok:
                                    failed, err = True, run.error
                                    break
                                c = (run.stats.sync_count, run.stats.words_reduced)
                                if counters is not None and c != counters:
                                    raise api.Error("bench: sync counters changed between "
                                                    "seeds for " + name)
                                counters = c
                                loos.append(run.loo)
                                ress.append(run.resid)
                                times.append(run.timing.factor_ms * 1e-3)
                            if failed:
                                exp = assumption_violated(name, kappa)
                                row.update(loo=math.nan, residual=math.nan,
                                           predicted_time=math.nan, failed=True,
                                           failure_expected=exp, error=err,
                                           measured_time=math.nan, gflops=math.nan)
                                row["speedup_vs_bcgsi+"] = math.nan
                                if not exp:
                                    rep.exit_code = 1
                                print(f"bench: cell ({name}, n={n}, m={m}, s={s}, "
                                      f"kappa={kappa:g}, P={procs}) aborted"
                                      f"{' (predicted by its stability assumption)' if exp else ' UNEXPECTEDLY'}"
                                      f": {err}", file=log)
                            else:
                                row["sync_count"], row["words_reduced"] = counters
                                t = predicted_time(cfg.alpha, cfg.beta, cfg.gamma, procs,
                                                   counters[0], counters[1], row["flops"])
                                if t <= 0 or t_base <= 0:
                                    raise ConfigError("predict_speedup: model predicts zero "
                                                      "time for a run")
                                tm = float(np.mean(times))
                                row.update(loo=float(np.mean(loos)), residual=float(np.mean(ress)),
                                           predicted_time=t, measured_time=tm,
                                           gflops=row["flops"] / tm / 1e9 if tm > 0 else math.nan)
                                row["speedup_vs_bcgsi+"] = t_base / t
                            rep.rows.append(row)
    return rep


def write_csv(rep: BenchReport, out) -> None:
    out.write(",".join(COLUMNS + EXTRA) + "\n")
    for r in rep.rows:
        vals = []
        for c in COLUMNS + EXTRA:
            v = r.get(c)
            vals.append(format_real(v) if isinstance(v, float) else str(v))
        out.write(",".join(vals) + "\n")


def write_json(rep: BenchReport, out) -> None:
    rows = []
    for r in rep.rows:
        d = {c: r[c] for c in COLUMNS}
        if r.get("failed"):
            d.update(failed=True, failure_expected=r["failure_expected"], error=r["error"])
        d.update({c: r.get(c) for c in EXTRA})
        rows.append(d)
    out.write(json.dumps(rows, indent=2, default=float) + "\n")


def emit(rep: BenchReport, path: str, fmt: str) -> int:
    if path:
        try:
            f = open(path, "w")
        except OSError:
            raise ConfigError(f"cannot open output file '{path}'") from None
    else:
        f = sys.stdout
    try:
        (write_json if fmt == "json" else write_csv)(rep, f)
    finally:
        if path:
            f.close()
    return rep.exit_code


# ---------------------------------------------------------------------------------------
# verify (verify_suite.cpp:43-194)
# ---------------------------------------------------------------------------------------
def _test_matrix(n, m, s, kappa, seed):
    return api.gen_matrix(n, m, s, kappa, seed, False)


def run_verify_suite(out=sys.stdout, ctx: Optional[api.Context] = None) -> int:
    ctx = ctx or api.default_context()
    names = [api.variant_name(v) for v in api.all_variants()]

    def sync_formulas():
        x = _test_matrix(64, 8, 2, 1e2, 7)
        for procs in (1, 3):
            for v in api.all_variants():
                run = api.run_factor(int(v), x, 2, procs, metrics=False, ctx=ctx)
                if not run.ok:
                    return f"{names[v]} aborted on a kappa=1e2 input: {run.error}"
                want = api.expected_syncs(int(v), 4)
                if run.stats.sync_count != want:
                    return (f"{names[v]} at q=4, P={procs}: expected {want} syncs, measured "
                            f"{run.stats.sync_count}")
        return None

    def single_block():
        x = _test_matrix(32, 4, 4, 1e2, 11)
        for v in api.all_variants():
            run = api.run_factor(int(v), x, 4, 2, metrics=False, ctx=ctx)
            if not run.ok:
                return f"{names[v]} aborted at q=1: {run.error}"
            if run.stats.sync_count != 1:
                return (f"{names[v]} at q=1 should cost exactly 1 sync, measured "
                        f"{run.stats.sync_count}")
        return None

    def transparency():
        x = _test_matrix(96, 8, 2, 1e2, 3)
        for v in (api.VariantId.BcgsIro, api.VariantId.BcgsIp1s):
            ref = api.run_factor(int(v), x, 2, 1, metrics=False, ctx=ctx)
            if not ref.ok:
                return f"{names[v]} aborted: {ref.error}"
            for procs in (2, 4):
                run = api.run_factor(int(v), x, 2, procs, metrics=False, ctx=ctx)
                if not run.ok:
                    return f"{names[v]} aborted: {run.error}"
                dq = np.abs(run.q - ref.q).max()
                dr = np.abs(run.r - ref.r).max() / np.abs(ref.r).max()
                if dq > 1e-13 or dr > 1e-13:
                    return (f"{names[v]}: Q / R differ between P=1 and P={procs} beyond "
                            f"rounding ({dq:.3g}, {dr:.3g})")
                if run.stats.sync_count != ref.stats.sync_count:
                    return f"{names[v]}: sync count depends on P"
        return None

    def quality():
        x = _test_matrix(128, 16, 4, 1e2, 19)
        for v in api.all_variants():
            run = api.run_factor(int(v), x, 4, 1, metrics=True, ctx=ctx)
            if not run.ok:
                return f"{names[v]} aborted on a kappa=1e2 input: {run.error}"
            if not run.loo <= 1e-10:
                return f"{names[v]}: loss of orthogonality {format_real(run.loo)} above 1e-10 at kappa=1e2"
            if not run.resid <= 1e-12:
                return f"{names[v]}: relative residual {format_real(run.resid)} above 1e-12"
            if np.any(np.tril(run.r, -1) != 0.0):
                return f"{names[v]}: R has a nonzero below the diagonal"
        return None

    def reprojection():
        x = _test_matrix(100, 16, 4, 1e3, 23)
        worst = [0.0]

        def probe(k, s2, q_local, x_local, shard):
            worst[0] = max(worst[0], float(np.abs(s2 - q_local.T @ x_local).max()))

        run = api.run_factor(int(api.VariantId.BcgsIp1s), x, 4, 1, metrics=False, ctx=ctx,
                             opts=api.BcgsOptions(probe=probe))
        if not run.ok:
            return "BCGSI+P-1S aborted: " + run.error
        if not worst[0] <= 1e-10:
            return "recurrence deviates from the direct product by " + format_real(worst[0])
        return None

    def speedup():
        q = 64

        def t(v):
            return predicted_time(1e-5, 0.0, 0.0, 1, api.expected_syncs(int(v), q), 0, 0.0)
        one = t(api.VariantId.BcgsIro) / t(api.VariantId.BcgsIp1s)
        two = t(api.VariantId.BcgsIro) / t(api.VariantId.BcgsIp2s)
        if not 3.9 <= one <= 4.0:
            return "one-sync speedup at q=64 out of band: " + format_real(one)
        if not 1.95 <= two <= 2.0:
            return "two-sync speedup at q=64 out of band: " + format_real(two)
        return None

    checks = [
        ("sync-count formulas (q=4, P in {1,3})", sync_formulas),
        ("single-block degenerate case costs 1 sync", single_block),
        ("distribution transparency (across P, to rounding: fp64 Gram on the GPU)", transparency),
        ("factorization quality at kappa=1e2", quality),
        ("delayed-reprojection identity", reprojection),
        ("speedup asymptotics at q=64", speedup),
    ]
    failures = 0
    for name, fn in checks:
        try:
            problem = fn()
        except Exception as e:  # noqa: BLE001
            problem = f"unexpected exception: {e}"
        if problem:
            failures += 1
            out.write(f"FAIL {name}: {problem}\n")
        else:
            out.write(f"PASS {name}\n")
    if failures:
        out.write(f"{failures} of {len(checks)} checks failed\n")
        return 1
    out.write(f"all {len(checks)} checks passed\n")
    return 0


# ---------------------------------------------------------------------------------------
# main (blockgs_main.cpp:93-146)
# ---------------------------------------------------------------------------------------
def _costs(p):
    p.add_argument("--cost-alpha", type=float, default=-1.0, help="Override: seconds per synchronization")
    p.add_argument("--cost-beta", type=float, default=-1.0, help="Override: seconds per word reduced")
    p.add_argument("--cost-gamma", type=float, default=-1.0, help="Override: seconds per flop per process")


def _apply_costs(a, cfg):
    for k in ("alpha", "beta", "gamma"):
        v = getattr(a, "cost_" + k)
        if v >= 0.0:
            setattr(cfg, k, v)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2507_21791_b200.cli",
                                 description="Block Gram-Schmidt factorization and sync-cost harness (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="Run a benchmark sweep described by a config file")
    b.add_argument("--config", required=True)
    _costs(b)
    f = sub.add_parser("factor", help="Factor one random test matrix and report")
    f.add_argument("--variant", required=True)
    f.add_argument("--n", type=int, required=True)
    f.add_argument("--m", type=int, required=True)
    f.add_argument("--s", type=int, required=True)
    f.add_argument("--kappa", type=float, default=1e2)
    f.add_argument("--seed", type=int, default=12345)
    f.add_argument("--procs", type=int, default=1)
    f.add_argument("--out", default="csv")
    f.add_argument("--distribution", default="geometric")
    _costs(f)
    sub.add_parser("verify", help="Run the built-in invariant suite")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "bench":
            cfg = parse_bench_config_file(a.config)
            _apply_costs(a, cfg)
            return emit(run_bench(cfg), cfg.out, cfg.format)
        if a.cmd == "factor":
            cfg = BenchConfig(variants=[int(api.parse_variant(a.variant))], n_values=[a.n],
                              m_values=[a.m], s_values=[a.s], kappa_values=[a.kappa],
                              procs_values=[a.procs], seeds=1, base_seed=a.seed)
            if a.distribution in ("gaussian", "random-gaussian"):
                cfg.distribution = "gaussian"
            elif a.distribution in ("geometric", "geometric-singular-values"):
                cfg.distribution = "geometric"
            else:
                raise ConfigError(f"unknown distribution '{a.distribution}'")
            if a.out not in ("csv", "json"):
                raise ConfigError("--out must be csv or json")
            cfg.format = a.out
            _apply_costs(a, cfg)
            return emit(run_bench(cfg), "", cfg.format)
        return run_verify_suite(sys.stdout)
    except api.ConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
