"""K7 partial attention + LSE merge, and the fused decode engine, on the GPU.

Tolerances: the kernels accumulate in f64 in the reference's order, so the
measured deviation is ~1e-15; the bar written here is the north star's fp32
bar of 1e-3 relative, tightened to 1e-9 where the computation is f64
end to end (documented per test)."""
import numpy as np
import pytest

from conftest import load_golden
from oracle.ffi import BuildParams

pytestmark = pytest.mark.gpu

F64_RTOL = 1e-9  # f64 accumulate on both sides; only exp() ulps and merge order differ


def _ra():
    import paper_2409_10516_b200 as ra
    return ra


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def test_partial_attention_matches_oracle(port):
    ra = _ra()
    rng = np.random.default_rng(21)
    for n, d in [(8, 4), (64, 8), (2048, 128), (300, 33)]:
        K = rng.standard_normal((n, d)).astype(np.float32)
        V = rng.standard_normal((n, d)).astype(np.float32)
        kv = ra.KVGroup(K, V)
        for m in (1, 5, min(n, 100), n):
            idx = rng.choice(n, size=m, replace=False).astype(np.uint32)
            q = rng.standard_normal(d).astype(np.float32)
            p = ra.partial_attention(q, kv, idx)
            o, zmax, expsum = port.partial_attention(q, K, V, idx)
            assert not p.empty
            assert p.zmax == zmax  # exact dot * inv_sqrt_d, max is order-free
            assert abs(p.expsum - expsum) <= 1e-12 * expsum
            assert rel(p.out, o) <= F64_RTOL


def test_partial_attention_single_index_and_errors():
    # test_attention.cpp:112-134, 238-253
    ra = _ra()
    rng = np.random.default_rng(6)
    K = rng.standard_normal((16, 8)).astype(np.float32)
    V = rng.standard_normal((16, 8)).astype(np.float32)
    kv = ra.KVGroup(K, V)
    q = rng.standard_normal(8).astype(np.float32)
    p = ra.partial_attention(q, kv, [11])
    np.testing.assert_allclose(p.out, V[11].astype(np.float64), rtol=1e-15)
    assert p.expsum == 1.0
    with pytest.raises(ra.InvalidArgument, match="empty index set"):
        ra.partial_attention(q, kv, [])
    with pytest.raises(ra.InvalidArgument, match="out of range"):
        ra.partial_attention(q, kv, [3, 16])
    with pytest.raises(ra.InvalidArgument, match="query dimension mismatch"):
        ra.partial_attention(q[:7], kv, [3])


def test_merge_reproduces_union_softmax(port):
    # test_attention.cpp:267-287: 200 random splits, rel <= 1e-5 vs direct softmax
    ra = _ra()
    rng = np.random.default_rng(31)
    for rep in range(50):
        K = rng.standard_normal((32, 8)).astype(np.float32)
        V = rng.standard_normal((32, 8)).astype(np.float32)
        q = rng.standard_normal(8).astype(np.float32)
        kv = ra.KVGroup(K, V)
        sel = rng.random(32) < 0.5
        w, o = np.where(sel)[0], np.where(~sel)[0]
        pw = ra.partial_attention(q, kv, w) if len(w) else ra.empty_partial(8)
        po = ra.partial_attention(q, kv, o) if len(o) else ra.empty_partial(8)
        gw, go = ra.merge_gammas(pw, po)
        assert abs(gw + go - 1.0) <= 1e-6
        merged = ra.merge(pw, po)
        z = (K.astype(np.float64) @ q.astype(np.float64)) / np.sqrt(8)
        e = np.exp(z - z.max())
        direct = (e[:, None] * V.astype(np.float64)).sum(0) / e.sum()
        assert rel(merged, direct) <= 1e-5
        ow = port.merge((pw.out, pw.zmax, pw.expsum) if not pw.empty else None,
                        (po.out, po.zmax, po.expsum) if not po.empty else None, 8)[0]
        assert rel(merged, ow) <= F64_RTOL


def test_merge_empty_sides():
    # test_attention.cpp:289-304
    ra = _ra()
    rng = np.random.default_rng(41)
    K = rng.standard_normal((16, 4)).astype(np.float32)
    V = rng.standard_normal((16, 4)).astype(np.float32)
    kv = ra.KVGroup(K, V)
    q = rng.standard_normal(4).astype(np.float32)
    pw = ra.partial_attention(q, kv, np.arange(16))
    out = ra.merge(pw, ra.empty_partial(4))
    np.testing.assert_array_equal(out, pw.out)
    assert ra.merge_gammas(pw, ra.empty_partial(4)) == (1.0, 0.0)
    with pytest.raises(ra.InvalidArgument, match="empty attention support"):
        ra.merge(ra.empty_partial(4), ra.empty_partial(4))


@pytest.mark.parametrize("name,h", [("d32", 0), ("d32", 1), ("d128", 0)])
def test_engine_matches_golden_run_head(name, h):
    """ra_engine_step (search -> partial W -> partial Omega -> merge) vs the
    reference's run_head pieces stored by make_golden.py."""
    import os
    from conftest import GOLDEN
    ra = _ra()
    w = load_golden(f"workload_{name}.npz")
    a = load_golden(f"attn_{name}_h{h}.npz")
    H, G = int(w["spec"][3]), int(w["spec"][4])
    g = h // (H // G)
    kv = ra.KVGroup(w["keys"][g], w["values"][g])
    with open(os.path.join(GOLDEN, f"graph_{name}_h{h}.oodg"), "rb") as f:
        graph = ra.OODGraph.from_blob(kv, f.read())
    eng = ra.Engine([kv], [graph], ra.EngineConfig(128, 512, 100, 128))
    for qi in range(len(a["out"])):
        out, om, sc = eng.decode_step(w["decode_q"][h][qi][None, :])
        ref_om = a["omega"][qi]
        np.testing.assert_array_equal(om[0], ref_om[: om.shape[1]])
        assert rel(out[0], a["out"][qi]) <= F64_RTOL


def test_engine_matches_reference_decode_step(port, ref, small_workload):
    """Whole decode_step (engine.cpp:105-115) against the reference engine on
    identical graphs: 4 heads, 2 GQA groups."""
    ra = _ra()
    w = small_workload
    bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
    blobs = [port.graph_build(w["keys"][h // 2], w["prefill_q"][h], bp) for h in range(4)]
    kvs = [ra.KVGroup(w["keys"][g], w["values"][g]) for g in range(2)]
    graphs = [ra.OODGraph.from_blob(kvs[h // 2], blobs[h]) for h in range(4)]
    for cfg in (ra.EngineConfig(128, 512, 100, None), ra.EngineConfig(16, 64, 50, 64),
                ra.EngineConfig(0, 0, 10, 32)):
        eng = ra.Engine(kvs, graphs, cfg)
        reng = ref.engine(w["keys"], w["values"], blobs, cfg.s_init, cfg.s_local, cfg.top_k,
                          -1 if cfg.search_param is None else cfg.search_param)
        for step in range(8):
            Q = np.stack([w["decode_q"][h][step] for h in range(4)])
            out, om, sc = eng.decode_step(Q)
            rout, rom, rsc = reng.step(Q, step)
            np.testing.assert_array_equal(om, rom[:, : om.shape[1]])
            np.testing.assert_array_equal(sc, rsc)
            for h in range(4):
                assert rel(out[h], rout[h]) <= F64_RTOL


def test_engine_window_covers_context(port):
    """t <= s_init + s_local: no retrieval, one partial over everything
    (test_engine.cpp:52-72)."""
    ra = _ra()
    wk = port.generate_workload(600, 64, 32, 2, 1, seed=7, n_decode=4)
    kv = ra.KVGroup(wk["keys"][0], wk["values"][0])
    blobs = [port.graph_build(wk["keys"][0], wk["prefill_q"][h], BuildParams(k_train=8,
                                                                            max_degree=4))
             for h in range(2)]
    graphs = [ra.OODGraph.from_blob(kv, b) for b in blobs]
    eng = ra.Engine([kv], graphs, ra.EngineConfig())
    Q = wk["decode_q"][:, 0, :]
    out, om, sc = eng.decode_step(Q)
    assert om.shape[1] == 0 and (sc == 0).all()
    for h in range(2):
        full, _, _ = port.partial_attention(Q[h], wk["keys"][0], wk["values"][0], np.arange(600))
        assert rel(out[h], full) <= F64_RTOL


def test_engine_rejects_malformed_setups(port, small_workload):
    # test_engine.cpp:280-307
    ra = _ra()
    w = small_workload
    kv = ra.KVGroup(w["keys"][0], w["values"][0])
    blob = port.graph_build(w["keys"][0], w["prefill_q"][0], BuildParams(k_train=8, max_degree=4))
    g = ra.OODGraph.from_blob(kv, blob)
    with pytest.raises(ra.InvalidArgument, match="top_k must be >= 1"):
        ra.Engine([kv], [g], ra.EngineConfig(top_k=0))
    eng = ra.Engine([kv], [g], ra.EngineConfig(top_k=100, search_param=50))
    with pytest.raises(ra.InvalidArgument, match="ef must be >= k"):
        eng.decode_step(w["decode_q"][0][:1])
    eng = ra.Engine([kv], [g], ra.EngineConfig())
    with pytest.raises(ra.InvalidArgument, match="one query per head required"):
        eng.decode_step(w["decode_q"][0][:2])


def test_engine_init_from_kvd1_workloads_matches_reference_engine(tmp_path, port):
    """Reference-style workloads (KVD1 round trip) -> engine_init on the GPU ->
    decode_step equals the oracle's run_head (engine.cpp:69-101)."""
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200 import kvd1
    from oracle.ffi import BuildParams
    w = port.generate_workload(1500, 64, 32, 4, 2, seed=11, n_decode=3)
    keys = [kvd1.VectorSet(1, w["keys"][g]) for g in range(2)]
    vals = [kvd1.VectorSet(2, w["values"][g]) for g in range(2)]
    heads = [kvd1.HeadWorkload(h, h // 2, kvd1.VectorSet(0, w["prefill_q"][h]), keys[h // 2],
                               vals[h // 2], kvd1.VectorSet(0, w["decode_q"][h]))
             for h in range(4)]
    kvd1.save_workloads(heads, 2, tmp_path)
    loaded = kvd1.load_workloads(tmp_path / "manifest.json")
    gp = ra.OODGraphBuildParams(32, 16, 64)
    eng = ra.engine_init(loaded, ra.EngineConfig(128, 512, 100, 128), gp)
    bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
    W = ra.static_partition(1500, 128, 512).static_set
    for step in range(3):
        Q = np.stack([w["decode_q"][h][step] for h in range(4)])
        out, omega, scanned = eng.decode_step(Q)
        for h in range(4):
            og = port.graph(w["keys"][h // 2], port.graph_build(w["keys"][h // 2],
                                                               w["prefill_q"][h], bp))
            r = og.search(Q[h], 100, W, 128)
            assert np.array_equal(omega[h], r.ids) and int(scanned[h]) == r.scanned
            pw = port.partial_attention(Q[h], w["keys"][h // 2], w["values"][h // 2], W)
            po = port.partial_attention(Q[h], w["keys"][h // 2], w["values"][h // 2], r.ids)
            ref = port.merge(pw, po, 32)[0]
            assert np.linalg.norm(out[h] - ref) / np.linalg.norm(ref) <= 1e-9


def test_engine_graph_replay_matches_eager(tmp_path):
    """RA_ENGINE_GRAPH=1 (whole-step CUDA graph) gives the same outputs as the
    eager launches, step after step (subprocess: the switch is read once)."""
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2409_10516_b200 as ra
from oracle.ffi import Oracle, BuildParams
port = Oracle("port")
w = port.generate_workload(2048, 64, 32, 2, 1, seed=9, n_decode=6)
bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
kv = ra.KVGroup(w["keys"][0], w["values"][0])
gs = [ra.OODGraph.from_blob(kv, port.graph_build(w["keys"][0], w["prefill_q"][h], bp)) for h in range(2)]
eng = ra.Engine([kv], gs, ra.EngineConfig(128, 512, 100, 128))
qh = torch.empty((2, 32), dtype=torch.float32, pin_memory=True)
out = torch.empty((2, 32), dtype=torch.float64, pin_memory=True)
om = torch.empty((2, 100), dtype=torch.int32, pin_memory=True)
sc = torch.empty(2, dtype=torch.int64, pin_memory=True)
res = []
for s in range(6):
    qh.copy_(torch.from_numpy(np.ascontiguousarray(w["decode_q"][:, s, :])))
    eng.ctx.bind_stream()
    ra.api._check(ra.lib.ra_engine_step_host(eng.h, qh.data_ptr(), out.data_ptr(), om.data_ptr(), sc.data_ptr()))
    res.append((out.clone().numpy(), om.clone().numpy(), sc.clone().numpy()))
np.save(sys.argv[1], np.array([np.concatenate([r[0].ravel(), r[1].ravel().astype(np.float64), r[2].astype(np.float64)]) for r in res]))
'''
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("0", "1"):
        f = tmp_path / f"r{flag}.npy"
        env = dict(os.environ, RA_ENGINE_GRAPH=flag)
        subprocess.run([sys.executable, "-c", code, str(f)], cwd=root, env=env, check=True)
        outs.append(np.load(f))
    np.testing.assert_array_equal(outs[0], outs[1])
