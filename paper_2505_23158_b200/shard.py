"""Multi-GPU view sharding.

Rendering shards naturally by camera view: a frame depends only on the
(replicated) store, its camera, its chunk pair and t, so ranks exchange
nothing on the data path.  Views are dealt block-cyclically: block b of
``block`` consecutive sweep views goes to rank ``b % world`` (contiguous
blocks keep the chunk pair mostly constant on a rank, cyclic dealing
balances cost along the path).  The only collectives gather per-rank
metrics and per-view results to rank 0 (NCCL over NVLink on B200, gloo in
the CPU tests), plus a max-over-ranks of the device-timed step.
"""

from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


def block_cyclic(n_views: int, world: int, rank: int, block: int = 16) -> List[List[int]]:
    """This rank's view blocks, in order (the last block may be short)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if block < 1:
        raise ValueError("block must be >= 1")
    n_blocks = -(-n_views // block)
    return [list(range(b * block, min((b + 1) * block, n_views)))
            for b in range(rank, n_blocks, world)]


def step_schedule(n_views: int, world: int, rank: int, n_steps: int,
                  block: int = 16) -> List[List[int]]:
    """Views per step for this rank: its blocks, cycling if n_steps exceeds them."""
    mine = block_cyclic(n_views, world, rank, block)
    if not mine:
        return [[] for _ in range(n_steps)]
    return [mine[s % len(mine)] for s in range(n_steps)]


def spread_schedule(n_views: int, world: int, rank: int, n_steps: int, block: int = 16,
                    offset: float = 0.5) -> List[List[int]]:
    """Views per step for this rank, spread over the whole sweep: step s takes
    this rank's block floor((s + offset) * n_mine / n_steps), so a short run
    samples the path evenly instead of its first blocks.  Distinct blocks
    whenever n_steps <= the rank's block count (cycling otherwise)."""
    mine = block_cyclic(n_views, world, rank, block)
    if not mine:
        return [[] for _ in range(n_steps)]
    if n_steps > len(mine):
        return [mine[s % len(mine)] for s in range(n_steps)]
    return [mine[min(len(mine) - 1, int((s + offset) * len(mine) / n_steps))]
            for s in range(n_steps)]


def max_over_ranks(value: float, device: Optional[torch.device] = None) -> float:
    """Max of a per-rank scalar (e.g. device-timed ms); identity without a group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(row: torch.Tensor) -> torch.Tensor:
    """all_gather of one fixed-size per-rank row -> (world, *row.shape)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return row.unsqueeze(0)
    out = [torch.zeros_like(row) for _ in range(dist.get_world_size())]
    dist.all_gather(out, row.contiguous())
    return torch.stack(out)


def gather_views(view_ids: torch.Tensor, payload: torch.Tensor, max_per_rank: int):
    """Gather variable-length per-view results (e.g. image checksums or 8-bit
    images) from all ranks: pads to ``max_per_rank`` rows, gathers, strips.

    Returns (view_ids, payload) concatenated over ranks, sorted by view id."""
    n = view_ids.shape[0]
    if n > max_per_rank:
        raise ValueError("more rows than max_per_rank")
    ids = torch.full((max_per_rank,), -1, dtype=torch.int64, device=view_ids.device)
    ids[:n] = view_ids
    pay = torch.zeros((max_per_rank,) + tuple(payload.shape[1:]), dtype=payload.dtype,
                      device=payload.device)
    pay[:n] = payload
    all_ids = gather_rows(ids).reshape(-1)
    all_pay = gather_rows(pay).reshape((-1,) + tuple(payload.shape[1:]))
    keep = all_ids >= 0
    all_ids, all_pay = all_ids[keep], all_pay[keep]
    order = torch.argsort(all_ids)
    return all_ids[order], all_pay[order]
