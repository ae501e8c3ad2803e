"""K6 graph search on the GPU vs the reference semantics.

Bar: bit-exact ids, f32 scores, scanned and truncated (the kernel runs the
reference's in-order f64 dot and reproduces the exact expanded set).
Graphs come from the oracle (golden OODG blobs and fresh oracle builds), so
these tests isolate the search from the builder.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle.ffi import BuildParams

pytestmark = pytest.mark.gpu


def _ra():
    import paper_2409_10516_b200 as ra
    return ra


def assert_same(a, b, ctx=""):
    np.testing.assert_array_equal(a.ids, b.ids, err_msg=ctx)
    np.testing.assert_array_equal(a.scores, b.scores, err_msg=ctx)
    assert a.scanned == b.scanned, ctx
    assert a.truncated == b.truncated, ctx


@pytest.mark.parametrize("name,h", [("d32", 0), ("d32", 1), ("d128", 0)])
def test_search_matches_golden(name, h):
    ra = _ra()
    w = load_golden(f"workload_{name}.npz")
    H, G = int(w["spec"][3]), int(w["spec"][4])
    kv = ra.KVGroup(w["keys"][h // (H // G)], w["values"][h // (H // G)])
    with open(os.path.join(GOLDEN, f"graph_{name}_h{h}.oodg"), "rb") as f:
        g = ra.OODGraph.from_blob(kv, f.read())
    W = ra.static_partition(int(w["spec"][0]), 128, 512).static_set
    s = load_golden(f"search_{name}_h{h}.npz")
    # batched: group rows by (mask, ef, k)
    for mi in (0, 1):
        for ef in np.unique(s["ef"]):
            sel = np.where((s["mask"] == mi) & (s["ef"] == ef))[0]
            k = int(s["k"][sel[0]])
            Q = w["decode_q"][h][s["qi"][sel]]
            res = ra.search_batch([g], Q, k, W if mi else None, int(ef)).host()
            for r, i in zip(res, sel):
                n = len(r.ids)
                np.testing.assert_array_equal(r.ids, s["ids"][i][:n])
                np.testing.assert_array_equal(r.scores, s["scores"][i][:n])
                assert r.scanned == s["scanned"][i]
                assert r.truncated == bool(s["truncated"][i])


def test_search_matches_oracle_random_graphs(port):
    ra = _ra()
    rng = np.random.default_rng(11)
    for n, d, M, nq in [(500, 16, 8, 100), (3000, 32, 16, 600), (1500, 128, 24, 300),
                        (700, 20, 12, 100), (64, 8, 32, 4)]:
        keys = rng.standard_normal((n, d)).astype(np.float32)
        tq = rng.standard_normal((nq, d)).astype(np.float32)
        blob = port.graph_build(keys, tq, BuildParams(k_train=min(32, n), max_degree=M,
                                                      ef_construction=2 * M))
        kv = ra.KVGroup(keys)
        g = ra.OODGraph.from_blob(kv, blob)
        og = port.graph(keys, blob)
        Q = rng.standard_normal((40, d)).astype(np.float32)
        mask = np.sort(rng.choice(n, size=n // 5, replace=False)).astype(np.uint32)
        for m in (None, mask):
            for ef, k in ((10, 10), (64, 20), (200, 100), (n, min(n, 300))):
                res = ra.search_batch([g], Q, k, m, ef).host()
                for qi in range(len(Q)):
                    assert_same(res[qi], og.search(Q[qi], k, m, ef), f"n={n} ef={ef} q={qi}")


def test_search_multi_graph_batch(port, small_workload):
    """One launch, several heads (graphs) and GQA-shared keys."""
    ra = _ra()
    w = small_workload
    bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
    kvs = [ra.KVGroup(w["keys"][g], w["values"][g]) for g in range(2)]
    graphs, ograph = [], []
    for h in range(4):
        blob = port.graph_build(w["keys"][h // 2], w["prefill_q"][h], bp)
        graphs.append(ra.OODGraph.from_blob(kvs[h // 2], blob))
        ograph.append(port.graph(w["keys"][h // 2], blob))
    W = ra.static_partition(2048, 128, 512).static_set
    for step in range(8):
        Q = np.stack([w["decode_q"][h][step] for h in range(4)])
        res = ra.search_batch(graphs, Q, 100, W, 128).host()
        for h in range(4):
            assert_same(res[h], ograph[h].search(Q[h], 100, W, 128), f"h={h} step={step}")


def line_graph(ra):
    # test_index_oodgraph.cpp:41-53 (hand-built geometry), graph from the oracle
    keys = np.array([[10, 0], [9, 0], [8, 0], [0, 5]], np.float32)
    return keys


def test_beam_search_walks_hand_built_graph(port):
    # test_index_oodgraph.cpp:113-140
    ra = _ra()
    keys = line_graph(ra)
    blob = port.graph_build(keys, np.array([[1, 0]], np.float32), BuildParams(k_train=3))
    g = ra.OODGraph.from_blob(ra.KVGroup(keys), blob)
    q = np.array([1, 0], np.float32)
    r = g.search(q, 2, None, 4)
    assert list(r.ids) == [0, 1] and abs(r.scores[0] - 10.0) < 1e-6
    assert r.scanned == 4 and not r.truncated
    m = g.search(q, 2, np.array([0], np.uint32), 4)
    assert list(m.ids) == [1, 2] and m.scanned == 4
    s = g.search(q, 1, None, 2)
    assert list(s.ids) == [0] and s.scanned == 4
    t = g.search(q, 10, None, 16)
    assert len(t.ids) == 4 and t.truncated


def test_search_parameter_validation(port):
    # test_index_oodgraph.cpp:384-400
    ra = _ra()
    rng = np.random.default_rng(71)
    keys = rng.standard_normal((32, 8)).astype(np.float32)
    blob = port.graph_build(keys, rng.standard_normal((8, 8)).astype(np.float32),
                            BuildParams(k_train=8, max_degree=4))
    g = ra.OODGraph.from_blob(ra.KVGroup(keys), blob)
    q = np.full(8, 0.5, np.float32)
    with pytest.raises(ra.InvalidArgument, match="^k must be >= 1$"):
        g.search(q, 0, None, 4)
    with pytest.raises(ra.InvalidArgument, match="^ef must be >= k$"):
        g.search(q, 5, None, 4)
    with pytest.raises(ra.InvalidArgument, match="^query dimension mismatch$"):
        g.search(np.full(7, 0.5, np.float32), 1, None, 4)


def test_single_key_graph(port):
    # test_index_oodgraph.cpp:402-412
    ra = _ra()
    keys = np.array([[0.3, -1.0, 2.0, 0.5]], np.float32)
    blob = port.graph_build(keys, keys, BuildParams())
    g = ra.OODGraph.from_blob(ra.KVGroup(keys), blob)
    assert g.entry_point() == 0 and g.reachable_count() == 1
    r = g.search(keys[0], 1, None, 1)
    assert list(r.ids) == [0]
    assert g.serialize() == blob


def test_blob_round_trip_and_malformed_blobs(port):
    # test_index_oodgraph.cpp:281-382
    ra = _ra()
    import struct
    keys2 = np.random.default_rng(61).standard_normal((2, 4)).astype(np.float32)
    kv = ra.KVGroup(keys2)
    good = b"OODG" + struct.pack("<IQIQ", 1, 2, 1, 0) + struct.pack("<IQ", 1, 1) + \
        struct.pack("<I", 0)
    assert list(ra.OODGraph.from_blob(kv, good).neighbors(0)) == [1]

    def expect(blob, msg):
        with pytest.raises(ra.GraphError, match="^" + msg + "$"):
            ra.OODGraph.from_blob(kv, blob)
    bad = b"X" + good[1:]
    expect(bad, "bad graph magic")
    expect(good[:4] + bytes([2]) + good[5:], "unsupported graph version")
    expect(b"OODG" + struct.pack("<IQ", 1, 3), "graph/key count mismatch")
    expect(good[:20] + bytes([9]) + good[21:], "entry point out of range")
    expect(b"OODG" + struct.pack("<IQIQ", 1, 2, 1, 0) + struct.pack("<IQQ", 2, 1, 1) +
           struct.pack("<I", 0), "degree exceeds bound")
    expect(good[:32] + bytes([7]) + good[33:], "neighbor id out of range")
    expect(good[:32] + bytes([0]) + good[33:], "self loop")
    expect(good + b"x", "trailing bytes in graph blob")
    expect(good[:-2], "truncated graph blob")

    rng = np.random.default_rng(51)
    keys = rng.standard_normal((512, 16)).astype(np.float32)
    blob = port.graph_build(keys, rng.standard_normal((128, 16)).astype(np.float32),
                            BuildParams(k_train=16, max_degree=8))
    g = ra.OODGraph.from_blob(ra.KVGroup(keys), blob)
    assert g.serialize() == blob
    assert g.memory_bytes() == 513 * 8 + (len(blob) - 28 - 4 * 512) // 8 * 4


def test_search_large_n_spills_and_global_visited(port):
    """A list that outgrows shared memory migrates to HBM; results unchanged.
    ef = n forces the whole graph through the candidate list."""
    ra = _ra()
    rng = np.random.default_rng(5)
    n, d = 20000, 16
    keys = rng.standard_normal((n, d)).astype(np.float32)
    blob = port.graph_build(keys, rng.standard_normal((64, d)).astype(np.float32),
                            BuildParams(k_train=8, max_degree=8, ef_construction=16))
    g = ra.OODGraph.from_blob(ra.KVGroup(keys), blob)
    og = port.graph(keys, blob)
    Q = rng.standard_normal((3, d)).astype(np.float32)
    res = ra.search_batch([g], Q, 100, None, n).host()
    for qi in range(3):
        r = og.search(Q[qi], 100, None, n)
        assert r.scanned == n
        assert_same(res[qi], r)


def test_search_throughput_mode_matches_oracle(port):
    """A batch larger than 2 x SMs takes the throughput-mode kernel (one
    query per warp): results must match the reference exactly too."""
    ra = _ra()
    rng = np.random.default_rng(23)
    n, d = 4000, 64
    keys = rng.standard_normal((n, d)).astype(np.float32)
    blob = port.graph_build(keys, rng.standard_normal((800, d)).astype(np.float32),
                            BuildParams(k_train=32, max_degree=24, ef_construction=64))
    g = ra.OODGraph.from_blob(ra.KVGroup(keys), blob)
    og = port.graph(keys, blob)
    B = 400  # > 2 x 148 SMs
    Q = rng.standard_normal((B, d)).astype(np.float32)
    mask = np.sort(rng.choice(n, size=300, replace=False)).astype(np.uint32)
    for m, ef, k in ((None, 64, 20), (mask, 128, 100)):
        res = ra.search_batch([g], Q, k, m, ef).host()
        for qi in range(0, B, 7):
            assert_same(res[qi], og.search(Q[qi], k, m, ef), f"tp ef={ef} q={qi}")


@pytest.mark.parametrize("kernel", ["lat", "tp", "tps", "tpr", "duo"])
def test_search_kernel_variants_identical(port, kernel):
    """Every K6 variant (latency CTA pipeline, throughput with shared-memory
    visited bits + TMA tiles, throughput with register rows) returns the
    oracle's ids / scores / scanned / truncated on a d=128 multi-head batch."""
    ra = _ra()
    n, H, G = 16384, 4, 2
    w = port.generate_workload(n, 256, 128, H, G, seed=9, n_decode=16)
    kvs = [ra.KVGroup(w["keys"][g], w["values"][g]) for g in range(G)]
    bp = ra.OODGraphBuildParams(32, 24, 128, 8)
    graphs = [ra.ood_build(kvs[h // 2], w["prefill_q"][h], bp) for h in range(H)]
    ograph = [port.graph(w["keys"][h // 2], graphs[h].serialize()) for h in range(H)]
    W = ra.static_partition(n, 128, 512).static_set
    ctx = ra.default_context()
    ctx.set_search_kernel(kernel)
    try:
        steps = 16
        Q = np.concatenate([np.stack([w["decode_q"][h][s] for h in range(H)])
                            for s in range(steps)])
        res = ra.search_batch(graphs * steps, Q, 100, W, 128).host()
        for i in range(len(res)):
            h = i % H
            assert_same(res[i], ograph[h].search(Q[i], 100, W, 128), f"{kernel} q={i}")
    finally:
        ctx.set_search_kernel(None)
