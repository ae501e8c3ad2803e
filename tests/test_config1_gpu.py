"""configs[0] end to end (single head, d=128, N=16K synthetic OOD keys and
queries, README graph parameters): the GPU build is byte-identical to the
REFERENCE's own ood_build, and 64 decode steps through decode_run produce
the reference's trace (ids, scanned) byte for byte."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.ffi import BuildParams, Oracle, available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")]


def test_config1_build_and_decode_identical_to_reference():
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.decode import decode_run
    from test_decode_gpu import _ref_run
    o = Oracle("ref")
    n, steps = 16384, 64
    w = o.generate_workload(n, 256, 128, 1, 1, seed=7, n_decode=steps,
                            n_threads=os.cpu_count())
    K, V, pq = w["keys"][0], w["values"][0], w["prefill_q"][0]
    ref_blob = o.graph_build(K, pq, BuildParams(k_train=128, max_degree=24, ef_construction=256,
                                                edge_window=8), n_threads=os.cpu_count())
    kv = ra.KVGroup(K, V)
    g = ra.ood_build(kv, pq, ra.OODGraphBuildParams(128, 24, 256, 8))
    assert g.serialize() == ref_blob
    eng = ra.Engine([kv], [g], ra.EngineConfig(128, 512, 100, 128))
    reng = o.engine(K[None], V[None], [ref_blob], 128, 512, 100, 128, os.cpu_count())
    ours = decode_run(eng, w["decode_q"], steps)
    rj, rs, _ = _ref_run(o, reng, w["decode_q"], steps, 0, 1, steps)
    assert ours.trace.to_jsonl(True) == rj
    assert ours.summary.to_json() == rs
