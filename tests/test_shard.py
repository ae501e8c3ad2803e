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


# ---------------------------------------------------------------------------
# the group split on real decode outputs: each rank runs the reference's own
# decode_step (oracle/_ref, engine.cpp:105-115) over ITS KV groups only, the
# outputs are all-gathered, and the result must equal the unsharded engine's
# bit for bit (heads are independent: engine.cpp:111)
# ---------------------------------------------------------------------------
def _engine_worker(rank, world, port, G, hpg, n, steps, q):
    import numpy as np
    from oracle.ffi import BuildParams, Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port_o, ref = Oracle("port"), Oracle("ref")
        w = port_o.generate_workload(n, 64, 32, G * hpg, G, seed=11, n_decode=steps)
        bp = BuildParams(k_train=16, max_degree=12, ef_construction=48)
        blobs = [port_o.graph_build(w["keys"][h // hpg], w["prefill_q"][h], bp)
                 for h in range(G * hpg)]
        groups = groups_for_rank(G, world, rank)
        heads = heads_for_groups(groups, hpg)
        gat = OutputGather(G, hpg, 32, world, rank, "cpu")
        if heads:
            eng = ref.engine(w["keys"][groups], w["values"][groups], [blobs[h] for h in heads],
                             16, 64, 24, 48, 1)
        full = ref.engine(w["keys"], w["values"], blobs, 16, 64, 24, 48, 1)
        ok = True
        for s in range(steps):
            qs = np.ascontiguousarray(w["decode_q"][:, s, :])
            local = (torch.from_numpy(eng.step(np.ascontiguousarray(qs[heads]), s)[0])
                     if heads else torch.zeros((0, 32), dtype=torch.float64))
            got = gat(local, dist)
            want = torch.from_numpy(full.step(qs, s)[0])
            ok = ok and bool(torch.equal(got, want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G", [4, 3])
def test_sharded_reference_engine_outputs_world2_gloo(G):
    from oracle.ffi import available
    if not (available("ref") and available("port")):
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    world, hpg = 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_engine_worker, args=(r, world, port, G, hpg, 1500, 3, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    results = [q.get(timeout=10) for _ in range(world)]
    assert all(ok for _, ok in results), results
