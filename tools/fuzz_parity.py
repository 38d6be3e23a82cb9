# Randomized parity fuzzing against the oracle: random (variant, n, m, s, procs, kappa,
# seed) within each variant's working assumption u kappa^p <= 1e-3 (p = 1 BCGSI+ / P-2S,
# 2 PIPI+ / P-1S, 3 BCGSI+1S; variant.cpp:88-104); R to 1e-10 (normwise), LOO / residual
# within 10x, identical sync accounting.  Optional BGS_POISON=1.  Prints failures.
#   python tools/fuzz_parity.py [count] [seed]
# FUZZ_NCCL=1: through bgs_factor_device on a one-rank NCCL context (the collective path;
# procs = 1) instead of bgs_factor.  FUZZ_PEER=1: the same on a one-rank peer-window context.
# FUZZ_DEVICE=1: the same on a plain one-GPU context (merged reduce + step, CUDA graphs).  In
# these device-path modes every fourth case runs two more matrices of its shape through the
# same buffers, so graphs are captured and replayed on new data.
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2507_21791_b200 as bgs
from oracle.oracle import Oracle
U = 2.0 ** -53
count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
o = Oracle()
import os
peer = os.environ.get("FUZZ_PEER") == "1"
dev = os.environ.get("FUZZ_DEVICE") == "1"  # bgs_factor_device on a plain one-GPU context
nccl = os.environ.get("FUZZ_NCCL") == "1" or peer or dev
if dev:
    import torch
    ctx = bgs.Context(0)
elif peer:
    # a one-rank peer context with the in-kernel wait: the step fused with the exchange
    # (reduce_xchg_step4_kernel) and the plain peer exchange on every other sync
    import torch
    ctx = bgs.Context(0, 0, 1, peer=True)
    ctx.peer_attach([ctx.peer_handle()], 2)
elif nccl:
    import torch
    ctx = bgs.Context(0, 0, 1, bgs.nccl_unique_id())
else:
    ctx = bgs.Context(0)


class _Out:
    pass


_bufs = {}


def factor_nccl(v, x, s):
    n, m = x.shape
    ld = (n + 31) // 32 * 32
    # fixed buffers per (m, ld): a repeated (variant, n, m, s) then has the signature of the
    # earlier call, so bgs_factor_device captures a CUDA graph on the second one and replays
    # it afterwards -- with different data each time (see the repeat step below)
    if (m, ld) not in _bufs:
        if len(_bufs) > 64:
            _bufs.clear()
        _bufs[(m, ld)] = (torch.zeros((m, ld), dtype=torch.float64, device="cuda"),
                          torch.zeros((m, ld), dtype=torch.float64, device="cuda"))
    X, Q = _bufs[(m, ld)]
    X.zero_()
    Q.zero_()
    X[:, :n] = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(x).T)).cuda()
    out = _Out()
    try:
        r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        out.ok, out.error, out.r, out.stats = True, "", r, st
        out.q = np.asfortranarray(Q[:, :n].cpu().numpy().T)
    except bgs.api.NotSpdError as e:
        out.ok, out.error = False, str(e)
    return out


fails, envelope, t0 = [], [], time.time()
for it in range(count):
    v = int(rng.integers(1, 6))
    s = int(rng.choice([1, 2, 3, 4, 4, 4, 5, 6, 8, 12, 16]))
    q = int(rng.integers(1, 13))
    m = s * q
    n = int(m + rng.integers(0, int(rng.choice([64, 4000, 30000]))))
    P = 1 if nccl else int(rng.choice([1, 1, 1, 2, 3, 5]))
    kappa = float(10.0 ** rng.uniform(0, 6))
    p = {1: 1, 2: 2, 3: 2, 4: 1, 5: 3}[v]
    if U * kappa ** p > 1e-3:
        continue
    gauss = bool(rng.integers(0, 2))
    seed = int(rng.integers(1, 10 ** 6))
    # device-path modes: every fourth case runs two more matrices of the same shape (other
    # seeds) through the same buffers: graph capture, then replay, on new data
    seeds = [seed]
    if nccl and it % 4 == 3:
        seeds += [seed + 1000003, seed + 2000003]
    for seed in seeds:
        x = o.gen_matrix(n, m, s, kappa, seed, gauss)
        ref = o.factor(v, x, s, P, metrics=True)
        if ref.rc != 0:
            continue
        try:
            out = factor_nccl(v, x, s) if nccl else bgs.run_factor(v, x, s, P, metrics=False, ctx=ctx)
        except Exception as e:  # noqa: BLE001
            fails.append((it, v, n, m, s, P, kappa, gauss, seed, "EXC " + str(e)[:60]))
            continue
        why = []
        if not out.ok:
            why.append("abort " + out.error[:50])
        else:
            mx = np.abs(ref.r).max()
            if np.abs(out.r - ref.r).max() > 1e-10 * mx:
                why.append("R %.1e" % (np.abs(out.r - ref.r).max() / mx))
            if out.stats.sync_count != ref.sync_count or out.stats.event_labels != ref.labels:
                why.append("syncs")
            loo, res = o.loo(out.q), o.residual(x, out.q, out.r)
            if loo > 10 * max(ref.loo, U):
                # The reference's own LOO depends on procs through the rounding of its tree and
                # sums (e.g. 1.3e-16 at P = 3 but 1.0e-15 .. 1.6e-15 at P = 1, 2, 4 on one case):
                # a value inside 10x of that envelope is reported apart, not as a failure.
                env_loo = max(o.factor(v, x, s, pp, metrics=True).loo for pp in (1, 2, 3, 4))
                if loo > 10 * max(env_loo, U):
                    why.append("loo %.1e vs %.1e (envelope %.1e)" % (loo, ref.loo, env_loo))
                else:
                    envelope.append((it, v, n, m, s, P, kappa, gauss, seed,
                                     "loo %.1e vs %.1e at P=%d, reference envelope over P=1..4 %.1e" % (loo, ref.loo, P, env_loo)))
            if res > 10 * max(ref.resid, U):
                why.append("res %.1e vs %.1e" % (res, ref.resid))
        if why:
            fails.append((it, v, n, m, s, P, kappa, gauss, seed, "; ".join(why)))
print(f"{count} cases in {time.time() - t0:.0f} s; failures: {len(fails)}"
      + (f"; {len(envelope)} LOO value(s) above 10x the same-P oracle but inside 10x of the reference's own envelope over P" if envelope else ""))
for f in fails:
    print("FAIL", f)
for f in envelope:
    print("ENVELOPE", f)
