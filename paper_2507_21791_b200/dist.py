"""One-process-per-GPU host plumbing (torch.distributed), replacing run_spmd's rank
threads and the communicator's rendezvous (communicator.hpp:98-152,
communicator.cpp:42-144) for a multi-GPU run.

torch.distributed (NCCL on GPUs, gloo in the CPU tests) is plumbing only: it moves the
NCCL unique id to every rank, gathers Q in rank order (gather_rows,
communicator.cpp:319-336), checks the replicated factors bitwise across ranks
(check_replication, runner.cpp:18-35) and takes max-over-ranks timings.  The per-step
collective of the algorithm itself is the NCCL allreduce issued by the C library on its
own stream (runtime.cu) -- or, for ranks that share one GPU (NCCL refuses two ranks on a
device), one ``host_allgather`` per sync through the library's host-communicator hook
(bgs_ctx_create_host_comm): the partials travel over torch.distributed (gloo) and are
summed in rank order by the library.
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


@dataclass
class RankInfo:
    rank: int
    world: int
    local_rank: int


def rank_info() -> RankInfo:
    return RankInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                    int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """distribute() ceil split (dist_block.cpp:37-43): rank owns [r*per, min((r+1)*per, n))."""
    per = (n + world - 1) // world
    r0 = min(rank * per, n)
    return r0, min(r0 + per, n) - r0


def exchange_unique_id(dist, rank: int, make_id: Callable[[], bytes]) -> bytes:
    """Rank 0 creates the ncclUniqueId; every rank receives the same 128 bytes."""
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad ncclUniqueId from rank 0")
    return bytes(uid)


def host_allgather(dist) -> Callable[[bytes], bytes]:
    """A blocking allgather of equal-size byte payloads over torch.distributed (the
    ``host_allgather`` of api.Context): returns every rank's payload concatenated in rank
    order (Communicator::rendezvous, communicator.cpp:96-144, over processes)."""
    import torch

    def allgather(payload: bytes) -> bytes:
        t = torch.frombuffer(bytearray(payload), dtype=torch.uint8)
        outs = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(outs, t)
        return b"".join(o.numpy().tobytes() for o in outs)
    return allgather


def attach_peers(dist, ctx, wait_mode: int = 0) -> None:
    """Exchange the window handles of a ``Context(peer=True)`` over torch.distributed and
    map every rank's window (bgs_ctx_peer_handle / bgs_ctx_peer_attach)."""
    handles = [None] * dist.get_world_size()
    dist.all_gather_object(handles, ctx.peer_handle())
    ctx.peer_attach(handles, wait_mode)
    dist.barrier()  # every window is mapped before anyone pushes


def gather_rows(dist, local: np.ndarray, n: int, world: int) -> np.ndarray:
    """Concatenate the ranks' row shards in rank order; every rank gets the n x m matrix
    (Communicator::gather_rows, communicator.cpp:319-336)."""
    import torch
    per = (n + world - 1) // world
    m = local.shape[1]
    pad = np.zeros((per, m))
    pad[: local.shape[0]] = local
    t = torch.from_numpy(pad)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    rows = []
    for r, o in enumerate(outs):
        _, cnt = shard_range(n, world, r)
        rows.append(o.numpy()[:cnt])
    return np.vstack(rows) if rows else np.zeros((0, m))


def digest(a: np.ndarray) -> bytes:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).digest()


def check_replication(dist, r: np.ndarray, what: str = "R") -> None:
    """Replicated factors must be bitwise identical on every rank (runner.cpp:18-35)."""
    mine = digest(r)
    allv = [None] * dist.get_world_size()
    dist.all_gather_object(allv, mine)
    for k, d in enumerate(allv):
        if d != allv[0]:
            raise RuntimeError(f"run_factor: replicated {what} differs between ranks 0 and {k}")


def max_over_ranks(dist, value: float) -> float:
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_factor_rank(dist, v: int, x_local, n: int, m: int, s: int,
                    ctx=None, device: Optional[int] = None):
    """Per-rank factorization of this rank's shard on its GPU (bcgs.hpp:49-50), then the
    reference's cross-rank replication check.  x_local: torch CUDA tensor (m, ld) holding
    the shard column-major.  Returns (R, stats, timing)."""
    import torch

    from . import api
    info = rank_info()
    dev = info.local_rank if device is None else device
    if ctx is None:
        uid = exchange_unique_id(dist, info.rank, api.nccl_unique_id) if info.world > 1 else None
        ctx = api.Context(dev, info.rank, info.world, uid)
    row0, nl = shard_range(n, info.world, info.rank)
    ld = x_local.shape[1]
    q_local = torch.zeros_like(x_local)
    r, st, tm = api.factor_device(ctx, v, n, m, s, row0, nl, x_local.data_ptr(), ld,
                                  q_local.data_ptr(), ld)
    if info.world > 1:
        check_replication(dist, r)
    return q_local, r, st, tm
