"""Host-side multi-GPU plumbing (torch.distributed only; no arithmetic of the method).

Rows of A shard naturally: r_i depends only on z_i = <a_i, x>,
so each rank holds a contiguous row block and F is the sum over ranks of the
local unnormalised sums, scaled by 1/n_global.  The library
does that sum with one ncclAllReduce per F evaluation; this module only
decides which rows a rank owns, ships the NCCL unique id from rank 0 to the
others, and reduces timings/byte counts for the benchmark.  Every function
works with any process-group backend (NCCL on the GPU box, gloo in the CPU
tests) — pass the device the backend expects.
"""
from __future__ import annotations

from dataclasses import replace


def row_block(n: int, rank: int, world: int) -> tuple[int, int]:
    """[row0, row1) of rank `rank` when n rows are split into `world`
    contiguous blocks whose sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError(f"bad shard request n={n} rank={rank} world={world}")
    return n * rank // world, n * (rank + 1) // world


def shard(cfg, rank: int, world: int, strong: bool):
    """(global config, row0, n_local, scaling) for this rank.

    strong: the config's n rows are split across ranks (total work fixed);
    weak: every rank holds the config's n rows of a problem `world` times
    larger (rows are keyed by global index, so the global problem is the same
    recipe with n*world rows)."""
    if world == 1:
        return cfg, 0, cfg.n, "strong" if strong else "weak"
    if strong:
        a, b = row_block(cfg.n, rank, world)
        return cfg, a, b - a, "strong"
    return replace(cfg, n=cfg.n * world), cfg.n * rank, cfg.n, "weak"


def exchange_id(make_id, rank: int, world: int) -> bytes | None:
    """Rank 0 calls make_id() (poly_nccl_unique_id) and broadcasts the bytes."""
    if world == 1:
        return None
    import torch.distributed as dist
    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def gather_handles(handle: bytes, rank: int, world: int) -> bytes:
    """All ranks' 64-byte peer-reduce window handles (poly_p2p_handle), in
    rank order, for poly_p2p_open (K9).  world == 1: the rank's own."""
    if len(handle) != 64:
        raise ValueError("a peer-reduce window handle is 64 bytes")
    if world == 1:
        return bytes(handle)
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, bytes(handle))
    if any(h is None or len(h) != 64 for h in out):
        raise RuntimeError("peer-reduce handle exchange incomplete")
    return b"".join(out)


def _reduce(value: float, op, device) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(value: float, world: int, device="cuda") -> float:
    """The benchmark's clock: the slowest rank's device time."""
    if world == 1:
        return float(value)
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.MAX, device)


def sum_over_ranks(value: float, world: int, device="cuda") -> float:
    if world == 1:
        return float(value)
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.SUM, device)
