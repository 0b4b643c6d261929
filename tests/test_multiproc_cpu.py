"""Multi-rank view sharding on CPU (gloo, world_size 2): the block-cyclic
schedule covers every view exactly once, max-over-ranks timing, and the
metric / per-view result gathers the bench uses on NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_23158_b200 import shard


def test_block_cyclic_covers_each_view_once():
    for world in (1, 2, 3, 4, 8):
        seen = []
        for r in range(world):
            for blk in shard.block_cyclic(4096, world, r, 16):
                assert len(blk) == 16 and blk == list(range(blk[0], blk[0] + 16))
                seen.extend(blk)
        assert sorted(seen) == list(range(4096))


def test_block_cyclic_ragged_and_errors():
    blocks = shard.block_cyclic(37, 2, 1, 16)
    assert blocks == [list(range(16, 32))]
    assert shard.block_cyclic(37, 2, 0, 16)[-1] == list(range(32, 37))
    with pytest.raises(ValueError):
        shard.block_cyclic(10, 2, 2)
    with pytest.raises(ValueError):
        shard.block_cyclic(10, 1, 0, 0)


def test_spread_schedule_covers_the_sweep():
    for world in (1, 2, 4, 8):
        steps = 20
        seen = []
        for r in range(world):
            sched = shard.spread_schedule(4096, world, r, steps, 16)
            assert len(sched) == steps
            firsts = [blk[0] for blk in sched]
            assert firsts == sorted(firsts) and len(set(firsts)) == steps
            seen.extend(v for blk in sched for v in blk)
        assert len(seen) == len(set(seen)) == steps * 16 * world
        # evenly spread: the sampled blocks reach both ends of the path
        assert min(seen) < 4096 // steps and max(seen) > 4096 - 4096 // steps - 16 * world


def test_step_schedule_cycles():
    s = shard.step_schedule(64, 4, 1, 5, 16)
    assert s[0] == list(range(16, 32)) and s[1] == s[0]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sched = shard.step_schedule(256, world, rank, 4, 16)
        mine = torch.tensor([v for blk in sched for v in blk], dtype=torch.int64)
        # per-view "result": a checksum-like row derived from the view id
        pay = torch.stack([mine.double() * 2.0, mine.double() + 0.5], dim=1)
        ids, rows = shard.gather_views(mine, pay, max_per_rank=64)
        ms = shard.max_over_ranks(10.0 + rank)
        metrics = shard.gather_rows(torch.tensor([float(rank), float(len(mine))]))
        q.put((rank, ids.tolist(), rows.tolist(), ms, metrics.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_gather_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ids, rows, ms, metrics in out:
        # 4 steps x 16 views per rank, disjoint blocks, all gathered in order
        assert ids == sorted(ids) and len(ids) == 128 and len(set(ids)) == 128
        assert all(r[0] == 2.0 * i and r[1] == i + 0.5 for i, r in zip(ids, rows))
        assert ms == 11.0
        assert metrics == [[0.0, 64.0], [1.0, 64.0]]
