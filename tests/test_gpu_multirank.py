"""Multi-rank runs on the one GPU this pool lends: P processes share cuda:0, each with its
own context and its own row shard, over two transports: the library's host-communicator
hook (bgs_ctx_create_host_comm) carried over torch.distributed gloo, and the one-shot
exchange over peer-mapped windows (bgs_ctx_create_peer: CUDA IPC between the processes,
stream memory operations for the wait).  NCCL refuses two ranks on
one device, and no kernel here waits on another rank (the exchange happens between
launches), so this is safe on a single GPU (B200_PROFILING.md: no cross-rank spinning).

What only runs with several real ranks is exercised: the per-step Gram allreduce, the
prologue's TSQR root allgather fused with its Gram allreduce (one sync), the cross-rank
TSQR tree with this rank's M offset, empty shards, and the reference's replication check
(runner.cpp:18-35): R must be bitwise identical on every rank.  Results are compared with
the oracle at the same procs (north_star tolerances) and the sync accounting is exact.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

U = 2.0 ** -53
# (variant, n, m, s, procs, kappa, gaussian)
CASES = [(v, 600, 32, 4, P, 1e3, False) for v in (1, 2, 3, 4, 5) for P in (2, 4)] + [
    (3, 1000, 48, 4, 8, 1e2, True),
    (5, 1000, 48, 4, 8, 1e2, True),
    (4, 301, 24, 3, 3, 1e4, False),     # ragged split, s = 3
    (3, 301, 24, 3, 3, 1e3, False),
    (1, 130, 64, 8, 4, 1e5, False),     # s = 8: the unfused K2t / K1 path
    (3, 12, 8, 4, 8, 1e1, True),        # ranks 6, 7 own no rows
    (2, 12, 8, 2, 8, 1e1, True),
    (3, 20000, 64, 4, 2, 1e6, False),   # the fused K12c path on each shard
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q, transport="host", env=None):
    os.environ.update(env or {})  # (runtime switches are read per call / per Runner)
    import torch
    import torch.distributed as dist

    import paper_2507_21791_b200 as bgs
    from oracle.oracle import Oracle
    from paper_2507_21791_b200 import dist as bd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        if transport == "peer":
            # one-shot exchange over CUDA-IPC windows; the ranks share cuda:0, so the
            # library waits with stream memory operations (no kernel spins on a rank)
            ctx = bgs.Context(0, rank, world, peer=True)
            bd.attach_peers(dist, ctx)
        else:
            ctx = bgs.Context(0, rank, world, host_allgather=bd.host_allgather(dist))
        for ci, (v, n, m, s, P, kappa, gauss) in enumerate(cases):
            if P != world:
                continue
            x = o.gen_matrix(n, m, s, kappa, 4242 + ci, gauss)
            r0, nl = bd.shard_range(n, world, rank)
            ld = max(32, (nl + 31) // 32 * 32)
            X = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
            if nl:
                X[:, :nl] = torch.from_numpy(np.ascontiguousarray(x[r0:r0 + nl].T)).cuda()
            Q = torch.zeros_like(X)
            try:
                r, st, _ = bgs.factor_device(ctx, v, n, m, s, r0, nl, X.data_ptr(), ld,
                                             Q.data_ptr(), ld)
                bd.check_replication(dist, r)
                qloc = Q[:, :nl].cpu().numpy().T.copy()
                q.put((ci, rank, "ok", r, qloc, st.sync_count, st.words_reduced,
                       list(st.event_labels)))
            except Exception as e:  # noqa: BLE001
                q.put((ci, rank, "err:" + str(e)[:300], None, None, 0, 0, []))
        q.put((-1, rank, "done", None, None, 0, 0, []))
    finally:
        dist.destroy_process_group()


def _run_world(world, transport="host", env=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q, transport, env))
             for r in range(world)]
    for p in procs:
        p.start()
    res, done = {}, 0
    try:
        while done < world:
            item = q.get(timeout=300)
            if item[0] < 0:
                done += 1
                continue
            res.setdefault(item[0], {})[item[1]] = item
    finally:
        for p in procs:  # a stuck rank must not outlive the test (exact PIDs we started)
            p.join(timeout=60 if done == world else 1)
            if p.is_alive():
                p.kill()
                p.join(timeout=10)
    for p in procs:
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("n_ranks,ng,ns", [(2, 16, 3000), (4, 0, 1), (8, 256, 26000), (3, 9, 100000)])
def test_peer_exchange_protocol_selftest(n_ranks, ng, ns):
    """The one-shot peer exchange (peer.cu) with emulated ranks in one process: every
    epoch all ranks push into all windows, then the spin flavour of the sum kernel runs
    with its flags already set.  Checked bitwise against the rank-ordered host sum on every
    rank, over both parities (bgs_peer_selftest)."""
    import paper_2507_21791_b200 as bgs
    bgs.peer_selftest(0, n_ranks, ng, ns, 6)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("transport", ["host", "peer"])
def test_ranks_sharing_one_gpu_match_oracle(oracle, world, transport):
    res = _run_world(world, transport)
    mine = [ci for ci, c in enumerate(CASES) if c[4] == world]
    assert sorted(res) == mine
    for ci in mine:
        v, n, m, s, P, kappa, gauss = CASES[ci]
        per = res[ci]
        assert sorted(per) == list(range(world))
        for rk in range(world):
            assert per[rk][2] == "ok", (CASES[ci], per[rk][2])
        x = oracle.gen_matrix(n, m, s, kappa, 4242 + ci, gauss)
        ref = oracle.factor(v, x, s, P, metrics=True)
        assert ref.rc == 0, ref.msg
        r0 = per[0][3]
        for rk in range(world):  # replicated R: bitwise identical on every rank
            assert np.array_equal(per[rk][3].view(np.int64), r0.view(np.int64))
            assert per[rk][5] == ref.sync_count and per[rk][6] == ref.words_reduced
            assert per[rk][7] == ref.labels
        q = np.vstack([per[rk][4] for rk in range(world)])
        mx = np.abs(ref.r).max()
        assert np.abs(r0 - ref.r).max() <= 1e-10 * mx, (CASES[ci], np.abs(r0 - ref.r).max() / mx)
        assert np.all(np.tril(r0, -1) == 0.0) and np.all(np.diag(r0) >= 0.0)
        loo, res_ = oracle.loo(q), oracle.residual(x, q, r0)
        assert loo <= 10 * max(ref.loo, U), (CASES[ci], loo, ref.loo)
        assert res_ <= 10 * max(ref.resid, U), (CASES[ci], res_, ref.resid)


def test_multirank_matches_emulated_procs(oracle):
    """The same factorization with 4 real ranks and with procs = 4 emulated on one
    context: same sync accounting, R within rounding of each other."""
    import paper_2507_21791_b200 as bgs
    res = _run_world(4)
    for ci, c in enumerate(CASES):
        if c[4] != 4:
            continue
        v, n, m, s, P, kappa, gauss = c
        x = oracle.gen_matrix(n, m, s, kappa, 4242 + ci, gauss)
        emu = bgs.run_factor(v, x, s, P, metrics=False)
        r = res[ci][0][3]
        assert np.abs(r - emu.r).max() <= 1e-12 * np.abs(emu.r).max()
        assert emu.stats.sync_count == res[ci][0][5]


@pytest.mark.parametrize("world", [2, 4])
def test_peer_fused_step_equals_separate_launches(world):
    """The one-sync step over the peer windows as two launches (reduce + push + flags, then
    rank-ordered sum + step: small.cu) against the same exchange as separate reduce / push /
    sum / step launches (BGS_NO_PEER_FUSE=1): same bits in R and Q on every rank, same
    sync accounting."""
    fused = _run_world(world, "peer")
    plain = _run_world(world, "peer", {"BGS_NO_PEER_FUSE": "1"})
    mine = [ci for ci, c in enumerate(CASES) if c[4] == world]
    assert sorted(fused) == mine and sorted(plain) == mine
    for ci in mine:
        for rk in range(world):
            a, b = fused[ci][rk], plain[ci][rk]
            assert a[2] == "ok" and b[2] == "ok", (CASES[ci], a[2], b[2])
            assert np.array_equal(a[3].view(np.int64), b[3].view(np.int64)), CASES[ci]
            assert np.array_equal(a[4].view(np.int64), b[4].view(np.int64)), CASES[ci]
            assert a[5:] == b[5:]


@pytest.mark.parametrize("one_launch", [1, 0])
@pytest.mark.parametrize("variant", [3, 5])
def test_peer_step_with_in_kernel_wait_on_one_rank(oracle, variant, one_launch, monkeypatch):
    """A one-rank peer context in the distinct-GPU mode (wait_mode 2: the flags are awaited
    inside the kernel).  one_launch = 1: reduce + push + flags + spin + sum + step in ONE
    kernel (reduce_xchg_step4_kernel); 0: two kernels, the second spinning at its head.
    With one rank the exchange is an identity, so R and Q must have the bits of the local
    (no-communicator) path, with fewer launches than the separate-launch exchange."""
    import torch

    import paper_2507_21791_b200 as bgs
    monkeypatch.setenv("BGS_PEER_ONE", str(one_launch))
    n, m, s = 20000, 64, 4
    x = oracle.gen_matrix(n, m, s, 1e4, 777, False)
    ld = (n + 31) // 32 * 32

    def run(ctx):
        X = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
        X[:, :n] = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        Q = torch.zeros_like(X)
        r, st, tm = bgs.factor_device(ctx, variant, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        return r, Q[:, :n].cpu().numpy(), st, tm

    local = run(bgs.Context(0))
    pctx = bgs.Context(0, 0, 1, peer=True)
    pctx.peer_attach([pctx.peer_handle()], 2)
    fused = run(pctx)
    monkeypatch.setenv("BGS_NO_PEER_FUSE", "1")
    plain = run(pctx)
    for other in (fused, plain):
        assert np.array_equal(local[0].view(np.int64), other[0].view(np.int64))
        assert np.array_equal(local[1].view(np.int64), other[1].view(np.int64))
        assert local[2].sync_count == other[2].sync_count
    steps = m // s - 2
    # separate launches: reduce, push, sum, step per block step; fused: 1 or 2
    assert plain[3].kernel_launches - fused[3].kernel_launches >= steps * (3 if one_launch else 2) - 4
