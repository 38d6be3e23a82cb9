#!/usr/bin/env python
"""Benchmark: fp64 BCGSI+P-1S QR on B200 (BASELINE.json metric / config 2).

One "step" = one full factorization X -> (Q, R) of the workload (default BASELINE
config 2: n=1e6, m=400, s=4, i.i.d. N(0,1)), rows sharded over the ranks, X resident in
HBM when the timed region starts.  `value` = whole-job fp64 GFLOP/s, the reference's own
analytic flop count (variant_flops, cost_model.cpp:29-119) / device time (max over ranks).

    python bench.py [--gpus N --steps K --warmup W]          # our B200 path
    python bench.py --impl reference [...]                   # the reference CPU path
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

VARIANT_DEFAULT = "BCGSI+P-1S"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default=VARIANT_DEFAULT)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--m", type=int, default=400)
    ap.add_argument("--s", type=int, default=4)
    ap.add_argument("--seed", type=int, default=12345)
    ap.add_argument("--dist", default="gaussian", choices=["gaussian", "geometric"],
                    help="i.i.d. N(0,1) (configs 1-4) or U diag(sigma) V^T (config 5)")
    ap.add_argument("--kappa", type=float, default=1e6, help="geometric: cond(X)")
    ap.add_argument("--config", type=int, default=0, choices=[0, 1, 2, 5],
                    help="BASELINE.json preset: 1 (n=1e5 m=64), 2 (n=1e6 m=400, the default "
                         "workload), 5 (n=1e7 m=400 geometric kappa=1e6)")
    ap.add_argument("--nccl", action="store_true",
                    help="N=1: run the collective path on a one-rank NCCL communicator")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="N>1: the per-step exchange over NCCL (default) or the library's one-shot "
                         "exchange over peer-mapped windows fused with the step kernel (NVLink P2P "
                         "stores, in-kernel wait; bgs_ctx_create_peer); N=1 with 'peer': a one-rank "
                         "peer context")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU seconds of one reference sample run")
    ap.add_argument("--ref-full", action="store_true",
                    help="--impl reference: time the whole workload once (no row sample)")
    a = ap.parse_args()
    if a.config == 1:
        a.n, a.m, a.s, a.dist = 100_000, 64, 4, "gaussian"
    elif a.config == 2:
        a.n, a.m, a.s, a.dist = 1_000_000, 400, 4, "gaussian"
    elif a.config == 5:
        a.n, a.m, a.s, a.dist, a.kappa = 10_000_000, 400, 4, "geometric", 1e6
    return a


def config_id(a):
    for cid, (n, m, s, dist) in {1: (100_000, 64, 4, "gaussian"), 2: (1_000_000, 400, 4, "gaussian"),
                                 5: (10_000_000, 400, 4, "geometric")}.items():
        if (a.n, a.m, a.s, a.dist) == (n, m, s, dist) and (dist == "gaussian" or a.kappa == 1e6):
            return f"BASELINE.json config {cid}"
    return "custom shape"


def dist_text(a):
    return ("i.i.d. N(0,1)" if a.dist == "gaussian"
            else f"U diag(sigma) V^T, sigma log-spaced 1..{1 / a.kappa:g}")


def workload_config(a, world):
    return {
        "workload": f"{a.variant} n={a.n} m={a.m} s={a.s} fp64 {dist_text(a)} ({config_id(a)})",
        "variant": a.variant, "n": a.n, "m": a.m, "s": a.s, "seed": a.seed,
        "dist": a.dist, **({"kappa": a.kappa} if a.dist == "geometric" else {}),
        "parallelism": f"row-sharded dp{world} (1-D ceil split), 1 allreduce per block step",
        "collectives": ("one-shot exchange over peer-mapped windows, fused with the step kernel"
                        if getattr(a, "transport", "nccl") == "peer" else
                        "NCCL" if world > 1 or getattr(a, "nccl", False)
                        else "none (one GPU: in-kernel reduction)"),
        "l2": f"inputs exceed L2: X is {a.n * a.m * 8 / 1e9:.2f} GB (126 MB L2), no flush needed",
    }


def metric_name(a):
    geo = "" if a.dist == "gaussian" else f" geometric kappa={a.kappa:.0e}".replace("+0", "")
    return f"fp64 QR time & GFLOP/s, {a.variant} n={a.n:.0e} m={a.m} s={a.s}{geo}".replace("+0", "")


# ---------------------------------------------------------------------------------------
# CPU reference (test-infrastructure checker, timed on the host cores)
# ---------------------------------------------------------------------------------------
def cpu_reference_runner(v, n, m, s, seed, gaussian=True, kappa=1.0):
    """Returns (kind, run(n_rows) -> (seconds, flops))."""
    from oracle.oracle import Oracle, Reference
    cores = os.cpu_count() or 1
    if Reference.available():
        ref = Reference()
        kind = "reference"

        def run(rows):
            x = ref.gen_matrix(rows, m, s, kappa if not gaussian else 1.0, seed, gaussian)
            res = ref.factor(v, x, s, procs=cores, want_q=False)
            return res.seconds
    else:
        ref = Oracle()
        kind = "port"
        cores = int(os.environ.get("OMP_NUM_THREADS", cores))

        def run(rows):
            x = ref.gen_matrix(rows, m, s, kappa if not gaussian else 1.0, seed, gaussian)
            t = time.perf_counter()
            ref.factor(v, x, s, 1)
            return time.perf_counter() - t
    return kind, cores, run


def pick_sample_rows(run, n, m, target_s):
    rows = max(m, 1000)
    t = run(rows)
    want = int(rows * target_s / max(t, 1e-3))
    return max(m, min(n, want)), t


# ---------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel):
    """dram bytes per launch / algorithmic bytes per launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel)
    except Exception:
        return None


# ---------------------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------------------
# VariantId order and canonical names of the reference (variant.hpp:8-15,
# variant.cpp:18-34); the reference arm resolves --variant with this table, not with our
# package (nothing of the product is loaded on this arm).
REF_VARIANTS = ["BCGS", "BCGSI+", "BCGSPIPI+", "BCGSI+P-1S", "BCGSI+P-2S", "BCGSI+1S"]


def run_reference_arm(a):
    """The reference's own CPU implementation (oracle/_ref, compiled from /root/reference
    by oracle/Makefile; the C port when it is absent) on this box's host cores, through
    its run_variant under run_spmd.  Each step is a bounded row sample of the workload
    (cost and flops are both linear in n); `value` is the measured GFLOP/s of those
    samples, `ms_per_step` their measured mean time -- nothing is extrapolated.
    --ref-full times the whole workload instead (config 2: ~6 min on 16 threads)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle.oracle import Oracle, Reference
    names = [x.upper() for x in REF_VARIANTS]
    if a.variant.upper() not in names:
        print(json.dumps({"impl": "reference", "unavailable": f"unknown variant {a.variant}"}))
        return 0
    v = names.index(a.variant.upper())
    counter = Reference() if Reference.available() else Oracle()
    per_step = max(2.0, a.cpu_seconds * 8.0 / max(8, a.steps + a.warmup))
    kind, cores, run = cpu_reference_runner(v, a.n, a.m, a.s, a.seed, a.dist == "gaussian",
                                            a.kappa)
    if a.ref_full:
        rows = a.n
        warm, steps = 0, 1
    else:
        rows, _ = pick_sample_rows(run, a.n, a.m, per_step)
        warm, steps = a.warmup, a.steps
    for _ in range(warm):
        run(rows)
    secs = [run(rows) for _ in range(steps)]
    t = sum(secs) / len(secs)
    flops = counter.variant_flops(v, rows, a.m, a.s)  # cost_model.cpp:29-119
    gf = flops / t / 1e9
    what = "the whole workload" if rows == a.n else "a row sample of the workload"
    sample = (f"{a.variant} n={rows} m={a.m} s={a.s} {dist_text(a)} ({what}; cost and flops "
              f"both linear in n), {'reference library oracle/_ref' if kind == 'reference' else 'oracle C port'} "
              f"run_variant under run_spmd with P={cores} threads, mean of {steps} timed runs "
              f"after {warm} warm-up runs")
    line = {
        "impl": "reference", "metric": metric_name(a), "value": gf, "unit": "GFLOP/s",
        "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded {dist_text(a)}, reference gen_matrix)",
        "config": workload_config(a, world),
        "sample_rows": rows,
        "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2507_21791_b200 as bgs
    from paper_2507_21791_b200 import api

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus if a.gpus == 1 else 1)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    uid = None
    if world > 1:
        obj = [bgs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    elif a.nccl:
        uid = bgs.nccl_unique_id()
    if a.transport == "peer":
        from paper_2507_21791_b200 import dist as bd
        ctx = bgs.Context(local, rank, world, peer=True)
        if world > 1:
            bd.attach_peers(dist, ctx, 2)  # distinct GPUs: the flags are awaited in the kernel
        else:
            ctx.peer_attach([ctx.peer_handle()], 2)
    else:
        ctx = bgs.Context(local, rank, world, uid)
    v = int(bgs.parse_variant(a.variant))
    n, m, s = a.n, a.m, a.s
    row0, nl = bgs.shard_rows(n, world, rank)
    ld = max(32, (nl + 31) // 32 * 32)  # tile engine reads whole 16-row blocks (bgs_gpu.h)
    X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
    Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    if a.dist == "gaussian":
        bgs.gen_gaussian_device(ctx, a.seed, row0, nl, m, X.data_ptr(), ld)
    else:  # config 5: U diag(sigma) V^T built on the GPUs (paper_2507_21791_b200/matgen.py)
        from paper_2507_21791_b200 import matgen
        matgen.geometric_device(ctx, n, m, a.kappa, a.seed, row0, nl, X, ld, scratch=Q)
        Q.zero_()
    torch.cuda.synchronize()
    flops = bgs.variant_flops(v, n, m, s)

    def step():
        return bgs.factor_device(ctx, v, n, m, s, row0, nl, X.data_ptr(), ld, Q.data_ptr(), ld)

    for _ in range(a.warmup):
        r, st, tm = step()
    barrier()
    torch.cuda.synchronize()
    ms_list, launches = [], 0
    with ClockSampler(local) as cs:
        t_wall = time.perf_counter()
        for _ in range(a.steps):
            r, st, tm = step()
            ms_list.append(tm.factor_ms)
            launches += tm.kernel_launches
        torch.cuda.synchronize()
        barrier()
        t_wall = time.perf_counter() - t_wall
    ms = allmax(sum(ms_list) / len(ms_list))
    value = flops / (ms * 1e-3) / 1e9
    # Per-kernel CUDA-event profile: the same steps again with every launch bracketed by
    # events on the library stream (kept out of the timed region above: the extra host
    # work per launch can open gaps between the short kernels).
    ctx.read_profile()
    ctx.profile(True)
    prof_ms = []
    for _ in range(a.steps):
        r, st, tm = step()
        prof_ms.append(tm.factor_ms)
    ctx.profile(False)
    prof = ctx.read_profile()

    # ---- roofline of the dominant kernel (live CUDA events over the timed region) ----
    peak, peak_src = hbm_peak()
    dom = max((k for k in prof if k in ("fused_update_gram", "gram", "update")),
              key=lambda k: prof[k]["ms"], default=None)
    roof = None
    kern = {}
    total_ms = sum(p["ms"] for p in prof.values())
    for k, p in prof.items():
        kern[k] = {"launches": p["launches"], "ms_total": p["ms"],
                   "share": p["ms"] / total_ms if total_ms else None,
                   "gbs": (p["alg_bytes"] / p["ms"] / 1e6) if p["ms"] and p["alg_bytes"] else None}
    if dom:
        p = prof[dom]
        ach = p["alg_bytes"] / p["ms"] / 1e6
        tr = ncu_traffic(dom)
        per_launch = p["alg_bytes"] / max(1, p["launches"])
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": (tr * per_launch) if tr else None, "kernel": dom,
                "peak_source": peak_src,
                "alg_bytes_per_launch": per_launch,
                "avg_launch_ms": p["ms"] / max(1, p["launches"])}
    # whole-factorization roofline: algorithmic bytes of all kernels / step time
    step_bytes = sum(p["alg_bytes"] for p in prof.values()) / a.steps
    prof_step_ms = sum(prof_ms) / len(prof_ms)

    # ---- verification at full size (untimed): LOO and residual on the device ----
    verify = None
    if not a.no_verify:
        loo, res = bgs.metrics_device(ctx, n, m, nl, X.data_ptr(), ld, Q.data_ptr(), ld, r)
        verify = {"loo": loo, "resid": res, "sync_count": st.sync_count,
                  "expected_syncs": bgs.expected_syncs(v, m // s),
                  "words_reduced": st.words_reduced}

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not a.no_e2e:
        hx = torch.empty((m, nl), dtype=torch.float64, pin_memory=True)
        hq = torch.empty((m, nl), dtype=torch.float64, pin_memory=True)
        hx.copy_(X[:, :nl])
        hr = np.zeros((m, m), order="F")
        st_, tm_, err_ = api._Stats(), api._Timing(), api._Err()
        dX = torch.empty((m, ld), dtype=torch.float64, device="cuda") if world > 1 else None

        def e2e_step():
            if world == 1:
                rc = api._lib.bgs_factor(ctx.handle, v, n, m, s, 1, hx.data_ptr(), nl,
                                         hq.data_ptr(), nl, hr.ctypes.data, m,
                                         ctypes.byref(st_), ctypes.byref(tm_), ctypes.byref(err_))
                api._raise(rc, err_)
            else:
                dX[:, :nl].copy_(hx, non_blocking=True)
                torch.cuda.synchronize()
                bgs.factor_device(ctx, v, n, m, s, row0, nl, dX.data_ptr(), ld, Q.data_ptr(), ld)
                hq.copy_(Q[:, :nl])
                torch.cuda.synchronize()

        e2e_step()
        barrier()
        ts = []
        for _ in range(max(1, a.steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t_e2e = allmax(sum(ts) / len(ts))
        e2e = {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s",
               "ms_per_step": t_e2e * 1e3,
               "h2d_bytes_per_step": n * m * 8, "d2h_bytes_per_step": n * m * 8 + m * m * 8 * world,
               "api": "bgs_factor (host X -> host Q, R; the run_factor drop-in)" if world == 1
               else "per rank: pinned H2D of the shard + bgs_factor_device + D2H of Q"}

    # ---- the same call from pageable host buffers (what a reference DenseMatrix caller has) ----
    e2e_pageable = None
    if not a.no_e2e and world == 1 and n * m * 8 <= 8e9:
        try:
            px = np.empty((m, nl), dtype=np.float64)
            px[...] = hx.numpy()
            pq = np.empty((m, nl), dtype=np.float64)
            pr = np.zeros((m, m), order="F")

            def pageable_step():
                rc = api._lib.bgs_factor(ctx.handle, v, n, m, s, 1, px.ctypes.data, nl, pq.ctypes.data, nl,
                                         pr.ctypes.data, m, ctypes.byref(st_), ctypes.byref(tm_),
                                         ctypes.byref(err_))
                api._raise(rc, err_)

            pageable_step()
            tp = []
            for _ in range(2):
                t0 = time.perf_counter()
                pageable_step()
                tp.append(time.perf_counter() - t0)
            t_pg = sum(tp) / len(tp)
            e2e_pageable = {"value": flops / t_pg / 1e9, "unit": "GFLOP/s", "ms_per_step": t_pg * 1e3,
                            "api": "bgs_factor from pageable numpy buffers (streamed through pinned rings)",
                            "same_bits_as_pinned": bool(np.array_equal(pq, hq.numpy()))}
            del px, pq
        except Exception as e:  # informational: never sinks the bench line
            e2e_pageable = {"value": None, "error": str(e)[:200]}

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        try:
            kind, cores, run = cpu_reference_runner(v, n, m, s, a.seed, a.dist == "gaussian",
                                                    a.kappa)
            rows, _ = pick_sample_rows(run, n, m, a.cpu_seconds)
            t = run(rows)
            gf = bgs.variant_flops(v, rows, m, s) / t / 1e9
            cpu = {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": kind,
                   "sample": f"{a.variant} n={rows} m={m} s={s} {dist_text(a)} (row subsample; cost and "
                             f"flops both linear in n), {t:.1f} s, run_variant under run_spmd "
                             f"with P={cores} threads",
                   "extrapolated_ms_full_n": t * 1e3 * n / rows}
        except Exception as e:  # the checker must never sink the bench line
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {e}"}

    clocks = cs.summary()
    if rank == 0:
        line = {
            "metric": metric_name(a), "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic: seeded i.i.d. N(0,1) generated on device (Philox)" if a.dist == "gaussian"
                     else "synthetic: X = U diag(sigma) V^T generated on device (U = QR of a Philox "
                          "Gaussian by this library, V host Haar, DGEMM)"),
            "config": workload_config(a, world),
            "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"],
                       "reasons": clocks["reasons"], "samples": clocks["samples"]},
            "e2e": e2e, "e2e_pageable": e2e_pageable, "gpu_launches": launches, "roofline": roof,
            "cpu_baseline": cpu,
            "time_ms": ms, "gflops": value,
            "step_roofline": {"alg_bytes": step_bytes, "achieved_gbs": step_bytes / ms / 1e6,
                              "frac": step_bytes / ms / 1e6 / peak},
            "kernels": kern, "profiled_pass_ms_per_step": prof_step_ms,
            "verify": verify, "wall_s_timed": t_wall,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference_arm(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
