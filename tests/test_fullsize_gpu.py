"""Parity at BASELINE.json's full size (configs[1]: 128K context, d=128,
README graph parameters): one KV group of the reference workload generated
on the GPU, four head graphs built by our builder, decode searches and the
whole decode step compared with the REFERENCE's own code (oracle/_ref) on
the same graphs (loaded through OODGraph(keys, blob)). Size-independent
properties are checked too: the OODG round trip is byte-stable, every node
is reachable from the entry, degrees respect the bound."""
import numpy as np
import pytest

from oracle.ffi import available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def layer():
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    spec = WorkloadSpec(n_ctx=131072, d_model=256, d_head=128, n_heads=32, n_kv_groups=8,
                        seed=7, n_decode=6)
    w = generate_group(spec, 3, "cuda")
    kv = ra.KVGroup(w["keys"], w["values"])
    bp = ra.OODGraphBuildParams(128, 24, 256, 8)
    graphs = [ra.ood_build(kv, w["prefill_q"][m], bp) for m in range(4)]
    return ra, kv, graphs, w["decode_q"].cpu().numpy(), w["keys"].cpu().numpy(), \
        w["values"].cpu().numpy()


def test_fullsize_graph_properties(layer):
    ra, kv, graphs, dq, K, V = layer
    for g in graphs:
        blob = g.serialize()
        assert ra.OODGraph.from_blob(kv, blob).serialize() == blob
        assert g.reachable_count() == 131072
        assert max(g.degree(u) for u in range(0, 131072, 997)) <= 24


def test_fullsize_search_and_step_match_reference(layer):
    ra, kv, graphs, dq, K, V = layer
    from oracle.ffi import Oracle
    o = Oracle("ref")
    W = ra.static_partition(131072, 128, 512).static_set
    og = [o.graph(K, g.serialize()) for g in graphs]
    eng = ra.Engine([kv], graphs, ra.EngineConfig(128, 512, 100, 128))
    reng = o.engine(K[None], V[None], [g.serialize() for g in graphs], 128, 512, 100, 128, 4)
    for step in range(dq.shape[1]):
        Q = np.ascontiguousarray(dq[:, step, :])
        # batched search (latency-mode kernel) == the reference's search
        res = ra.search_batch(graphs, Q, 100, W, 128).host()
        for h in range(4):
            r = og[h].search(Q[h], 100, W, 128)
            np.testing.assert_array_equal(res[h].ids, r.ids)
            np.testing.assert_array_equal(res[h].scores, r.scores)
            assert res[h].scanned == r.scanned and res[h].truncated == r.truncated
        # the whole decode step == the reference's decode_step
        out, om, sc = eng.decode_step(Q)
        rout, rom, rsc = reng.step(Q, step)
        np.testing.assert_array_equal(om, rom[:, : om.shape[1]])
        np.testing.assert_array_equal(sc, rsc)
        rel = np.linalg.norm(out - rout, axis=1) / np.linalg.norm(rout, axis=1)
        assert rel.max() <= 1e-12, rel


def test_fullsize_build_blob_identical_to_reference_ood_build():
    """configs[1]'s graph build at full size: the REFERENCE's own ood_build
    (oracle/_ref, all host threads) and our GPU build on the same 128K head
    (reference generator, seed 7, README parameters) write the same OODG
    bytes (kNN lists, projection, prune, entry point and repair)."""
    import os
    import paper_2409_10516_b200 as ra
    from oracle.ffi import BuildParams, Oracle
    o = Oracle("ref")
    n = 131072
    w = o.generate_workload(n, 256, 128, 1, 1, seed=7, n_decode=1, n_threads=os.cpu_count())
    keys, pq = w["keys"][0], w["prefill_q"][0]
    ref_blob = o.graph_build(keys, pq, BuildParams(128, 24, 256, 8), n_threads=os.cpu_count())
    kv = ra.KVGroup(keys, w["values"][0])
    g = ra.ood_build(kv, pq, ra.OODGraphBuildParams(128, 24, 256, 8))
    assert g.serialize() == ref_blob


def test_256k_search_identical_to_reference():
    """256K context (between configs[1] and configs[4]): GPU-built graph,
    eight masked searches on the GPU vs the reference's search on the same
    graph: identical ids, f32 scores, scanned and truncated."""
    import paper_2409_10516_b200 as ra
    from oracle.ffi import Oracle
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    n = 262144
    spec = WorkloadSpec(n_ctx=n, d_model=256, d_head=128, n_heads=32, n_kv_groups=8,
                        seed=11, n_decode=8)
    w = generate_group(spec, 5, "cuda")
    kv = ra.KVGroup(w["keys"], w["values"])
    g = ra.ood_build(kv, w["prefill_q"][1], ra.OODGraphBuildParams(128, 24, 256, 8))
    K = w["keys"].cpu().numpy()
    Q = w["decode_q"][1].cpu().numpy()
    W = ra.static_partition(n, 128, 512).static_set
    og = Oracle("ref").graph(K, g.serialize())
    res = ra.search_batch([g], Q, 100, W, 128).host()
    for i in range(Q.shape[0]):
        r = og.search(Q[i], 100, W, 128)
        np.testing.assert_array_equal(res[i].ids, r.ids)
        np.testing.assert_array_equal(res[i].scores, r.scores)
        assert res[i].scanned == r.scanned and res[i].truncated == r.truncated
