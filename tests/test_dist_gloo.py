"""N>1 host logic on CPU: world-size-2 gloo process groups exercise the rank plumbing of
paper_2507_21791_b200/dist.py (unique-id exchange, rank-ordered gather_rows, bitwise
replication check, max-over-ranks) and its agreement with the library's ceil split."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, q):
    import torch.distributed as dist

    from paper_2507_21791_b200 import dist as bd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        x = rng.standard_normal((n, m))
        r0, rows = bd.shard_range(n, world, rank)
        full = bd.gather_rows(dist, x[r0:r0 + rows], n, world)
        ok_gather = np.array_equal(full, x)
        uid = bd.exchange_unique_id(dist, rank, lambda: bytes(range(128)))
        ok_uid = uid == bytes(range(128))
        rmat = np.triu(np.ones((m, m)))
        bd.check_replication(dist, rmat)
        bad = rmat.copy()
        if rank == 1:
            bad[0, 0] = np.nextafter(1.0, 2.0)
        try:
            bd.check_replication(dist, bad)
            ok_detect = False
        except RuntimeError as e:
            ok_detect = "differs between ranks 0 and 1" in str(e)
        mx = bd.max_over_ranks(dist, 10.0 + rank)
        q.put((rank, ok_gather, ok_uid, ok_detect, mx, (r0, rows)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 7, 1])
def test_world2_rank_plumbing(n):
    import paper_2507_21791_b200 as bgs
    world, m = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_gather, ok_uid, ok_detect, mx, shard in res:
        assert ok_gather and ok_uid and ok_detect
        assert mx == 11.0
        assert shard == bgs.shard_rows(n, world, rank)


def _ag_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2507_21791_b200 import dist as bd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ag = bd.host_allgather(dist)
        payload = np.arange(5, dtype=np.float64) + 100 * rank
        out = np.frombuffer(ag(payload.tobytes()), dtype=np.float64).reshape(world, 5)
        # the library sums the gathered partials in rank order: identical bits everywhere
        tot = out[0].copy()
        for r in range(1, world):
            tot = tot + out[r]
        q.put((rank, out.tolist(), tot.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_allgather_rank_order(world):
    """dist.host_allgather (the host-communicator transport of bgs_ctx_create_host_comm):
    every rank receives all payloads in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ag_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [[float(i + 100 * r) for i in range(5)] for r in range(world)]
    for _, out, _ in res:
        assert out == want
    assert len({t for _, _, t in res}) == 1
