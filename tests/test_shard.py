"""Sharding by KV group and the output all_gather, on CPU with gloo
(world_size 2, two processes on 127.0.0.1)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_10516_b200.shard import (OutputGather, groups_for_rank, heads_for_groups,
                                         max_local_heads)


@pytest.mark.parametrize("G,world", [(8, 1), (8, 2), (8, 3), (8, 4), (8, 8), (2, 2), (5, 4)])
def test_groups_partition_is_a_balanced_cover(G, world):
    parts = [groups_for_rank(G, world, r) for r in range(world)]
    flat = [g for p in parts for g in p]
    assert flat == list(range(G))                      # contiguous, ordered, complete
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1
    hpg = 4
    heads = [h for p in parts for h in heads_for_groups(p, hpg)]
    assert heads == list(range(G * hpg))
    assert max_local_heads(G, world, hpg) == max(sizes) * hpg


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, G, hpg, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        groups = groups_for_rank(G, world, rank)
        heads = heads_for_groups(groups, hpg)
        # per-head "decode outputs": a deterministic function of the head id
        local = torch.stack([torch.full((d,), float(h), dtype=torch.float64) + torch.arange(d)
                             for h in heads]) if heads else torch.zeros((0, d), dtype=torch.float64)
        gat = OutputGather(G, hpg, d, world, rank, "cpu")
        for step in range(3):  # buffers reused across steps
            out = gat(local + step, dist)
            want = torch.stack([torch.full((d,), float(h), dtype=torch.float64) + torch.arange(d)
                                for h in range(G * hpg)]) + step
            q.put((rank, step, bool(torch.equal(out, want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G", [8, 3])
def test_output_all_gather_world2_gloo(G):
    world, hpg, d = 2, 4, 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, G, hpg, d, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = [q.get(timeout=10) for _ in range(world * 3)]
    assert all(ok for _, _, ok in results), results
