"""bf16 KV groups: the decode path reads bf16 rows. Bar: identical to the
reference run on the bf16-rounded K/V (ids, scores, scanned exact; output
within 1e-12), and within the north star's 1e-2 relative of the f32 output."""
import numpy as np
import pytest

from oracle.ffi import BuildParams

pytestmark = pytest.mark.gpu


def bf16_round(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("d", [128, 64, 32])
def test_bf16_search_and_step_equal_reference_on_rounded_kv(port, d):
    import paper_2409_10516_b200 as ra
    n, H = 3000, 2
    w = port.generate_workload(n, 256, d, H, 1, seed=13, n_decode=4)
    K, V = w["keys"][0], w["values"][0]
    Kr, Vr = bf16_round(K), bf16_round(V)
    kv = ra.KVGroup(K, V, dtype="bf16")
    np.testing.assert_array_equal(kv.keys_tensor().cpu().numpy(), Kr)
    bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
    blobs = [port.graph_build(Kr, w["prefill_q"][h], bp) for h in range(H)]
    graphs = [ra.OODGraph.from_blob(kv, b) for b in blobs]
    g_gpu = ra.ood_build(kv, w["prefill_q"][0], ra.OODGraphBuildParams(32, 16, 64))
    assert g_gpu.serialize() == blobs[0]   # the builder sees the rounded keys
    W = ra.static_partition(n, 128, 512).static_set
    eng = ra.Engine([kv], graphs, ra.EngineConfig(128, 512, 100, 128))
    kv32 = ra.KVGroup(K, V)
    eng32 = ra.Engine([kv32], [ra.OODGraph.from_blob(kv32, b) for b in blobs],
                      ra.EngineConfig(128, 512, 100, 128))
    for step in range(4):
        Q = np.stack([w["decode_q"][h][step] for h in range(H)])
        res = ra.search_batch(graphs, Q, 100, W, 128).host()
        out, om, sc = eng.decode_step(Q)
        out32, _, _ = eng32.decode_step(Q)
        for h in range(H):
            og = port.graph(Kr, blobs[h])
            r = og.search(Q[h], 100, W, 128)
            np.testing.assert_array_equal(res[h].ids, r.ids)
            np.testing.assert_array_equal(res[h].scores, r.scores)
            assert res[h].scanned == r.scanned
            assert np.array_equal(om[h], r.ids) and int(sc[h]) == r.scanned
            pw = port.partial_attention(Q[h], Kr, Vr, W)
            po = port.partial_attention(Q[h], Kr, Vr, r.ids)
            ref = port.merge(pw, po, d)[0]
            assert np.linalg.norm(out[h] - ref) / np.linalg.norm(ref) <= 1e-12
            assert np.linalg.norm(out[h] - out32[h]) / np.linalg.norm(out32[h]) <= 1e-2


def test_bf16_throughput_mode_batch(port):
    """a batch above 2 x SMs runs the throughput-mode kernel on bf16 rows"""
    import paper_2409_10516_b200 as ra
    rng = np.random.default_rng(4)
    n, d = 4000, 128
    K = rng.standard_normal((n, d)).astype(np.float32)
    Kr = bf16_round(K)
    blob = port.graph_build(Kr, rng.standard_normal((800, d)).astype(np.float32),
                            BuildParams(k_train=32, max_degree=24, ef_construction=64))
    g = ra.OODGraph.from_blob(ra.KVGroup(K, dtype="bf16"), blob)
    og = port.graph(Kr, blob)
    Q = rng.standard_normal((400, d)).astype(np.float32)
    res = ra.search_batch([g], Q, 50, None, 64).host()
    for qi in range(0, 400, 11):
        r = og.search(Q[qi], 50, None, 64)
        np.testing.assert_array_equal(res[qi].ids, r.ids)
        assert res[qi].scanned == r.scanned


def test_bf16_attention_only_keeps_ids_and_meets_tolerance(port):
    """bf16_attn: exact f32 search (ids identical to the f32 engine), bf16 K/V
    in the sparse attention: output within the north star's 1e-2 of f32."""
    import paper_2409_10516_b200 as ra
    n, H, d = 4000, 4, 128
    w = port.generate_workload(n, 256, d, H, 2, seed=21, n_decode=4)
    bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
    blobs = [port.graph_build(w["keys"][h // 2], w["prefill_q"][h], bp) for h in range(H)]
    mk = lambda dt: [ra.KVGroup(w["keys"][g], w["values"][g], dtype=dt) for g in range(2)]
    k32, kb = mk("f32"), mk("bf16_attn")
    e32 = ra.Engine(k32, [ra.OODGraph.from_blob(k32[h // 2], b) for h, b in enumerate(blobs)],
                    ra.EngineConfig(128, 512, 100, 128))
    eb = ra.Engine(kb, [ra.OODGraph.from_blob(kb[h // 2], b) for h, b in enumerate(blobs)],
                   ra.EngineConfig(128, 512, 100, 128))
    for step in range(4):
        Q = np.stack([w["decode_q"][h][step] for h in range(H)])
        o32, om32, sc32 = e32.decode_step(Q)
        ob, omb, scb = eb.decode_step(Q)
        np.testing.assert_array_equal(omb, om32)
        np.testing.assert_array_equal(scb, sc32)
        rel = np.linalg.norm(ob - o32, axis=1) / np.linalg.norm(o32, axis=1)
        assert rel.max() <= 1e-2, rel
