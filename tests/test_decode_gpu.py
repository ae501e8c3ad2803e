"""decode_run / trace / summary (engine.cpp:117-182) on the GPU vs the
reference's own decode_run (oracle/_ref) on the same graphs: trace JSONL and
summary JSON byte-identical; with compute_reference, mse at exp()-noise level."""
import ctypes as C

import numpy as np
import pytest

from oracle.ffi import REF_LIB, BuildParams, Oracle, available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")]


def _ref_run(o, reng, dq, n_steps, compute_reference, include_omega, n_entries):
    lib = o.lib
    f = lib.ref_engine_run
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_char_p, C.c_uint64,
                  C.POINTER(C.c_uint64), C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64),
                  C.c_void_p]
    l1, l2 = C.c_uint64(), C.c_uint64()
    dq = np.ascontiguousarray(dq, np.float32)
    mse = np.zeros(n_entries, np.float64)
    assert f(reng.h, dq.ctypes.data, n_steps, compute_reference, include_omega, None, 0,
             C.byref(l1), None, 0, C.byref(l2), None) == 0
    b1, b2 = C.create_string_buffer(l1.value + 1), C.create_string_buffer(l2.value + 1)
    assert f(reng.h, dq.ctypes.data, n_steps, compute_reference, include_omega, b1, l1.value,
             C.byref(l1), b2, l2.value, C.byref(l2), mse.ctypes.data) == 0
    return b1.raw[: l1.value].decode(), b2.raw[: l2.value].decode(), mse


def test_decode_run_matches_reference(port):
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.decode import decode_run, engine_memory
    o = Oracle("ref")
    n, H, G, steps = 3000, 4, 2, 5
    w = port.generate_workload(n, 64, 32, H, G, seed=5, n_decode=steps)
    bp = BuildParams(k_train=32, max_degree=16, ef_construction=64)
    blobs = [port.graph_build(w["keys"][h // 2], w["prefill_q"][h], bp) for h in range(H)]
    kvs = [ra.KVGroup(w["keys"][g], w["values"][g]) for g in range(G)]
    graphs = [ra.OODGraph.from_blob(kvs[h // 2], blobs[h]) for h in range(H)]
    eng = ra.Engine(kvs, graphs, ra.EngineConfig(128, 512, 100, 128))
    reng = o.engine(w["keys"], w["values"], blobs, 128, 512, 100, 128, 4)
    for inc in (0, 1):
        ours = decode_run(eng, w["decode_q"], steps)
        rj, rs, _ = _ref_run(o, reng, w["decode_q"], steps, 0, inc, H * steps)
        assert ours.trace.to_jsonl(bool(inc)) == rj
        assert ours.summary.to_json() == rs
    ours = decode_run(eng, w["decode_q"], steps, compute_reference=True)
    rj, rs, rmse = _ref_run(o, reng, w["decode_q"], steps, 1, 0, H * steps)
    mine = np.array([e.mse for e in ours.trace.entries])
    # mse compares two vectors that agree to ~1e-11 (the sparse result holds
    # nearly all attention mass): their difference is at the level of exp()'s
    # last-ulp noise (device vs libm), so agreement is absolute, not relative
    scale = max(1.0, float(np.max(np.abs(rmse))))
    np.testing.assert_allclose(mine, rmse, rtol=1e-2, atol=1e-18 * scale)
    assert mine.max() > 0
    kv_bytes, idx_bytes = engine_memory(eng)
    assert kv_bytes == G * n * 32 * 4 * 2
    assert idx_bytes == sum(g.memory_bytes() for g in graphs)


def test_decode_run_needs_enough_queries(port):
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.decode import decode_run
    w = port.generate_workload(1000, 64, 32, 1, 1, seed=3, n_decode=2)
    kv = ra.KVGroup(w["keys"][0], w["values"][0])
    g = ra.OODGraph.from_blob(kv, port.graph_build(w["keys"][0], w["prefill_q"][0],
                                                    BuildParams(k_train=16, max_degree=8)))
    eng = ra.Engine([kv], [g], ra.EngineConfig(128, 512, 100, 128))
    with pytest.raises(ra.InvalidArgument, match="^insufficient decode queries$"):
        decode_run(eng, w["decode_q"], 3)
