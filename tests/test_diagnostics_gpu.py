"""recall_sweep (diagnostics.cpp:143-194) on the GPU indexes vs the
reference's own indexes (oracle/_ref ref_recall_sweep, a restatement over
the unmodified library): CSV and JSONL reports byte-identical for flat,
ivf and oodgraph, plus the reference's errors."""
import ctypes as C

import numpy as np
import pytest

from oracle.ffi import REF_LIB, Oracle, available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def head():
    from paper_2409_10516_b200 import kvd1
    w = Oracle("ref").generate_workload(3000, 64, 32, 1, 1, seed=7, n_decode=24)
    return kvd1.HeadWorkload(0, 0, kvd1.VectorSet(0, w["prefill_q"][0]),
                             kvd1.VectorSet(1, w["keys"][0]), kvd1.VectorSet(2, w["values"][0]),
                             kvd1.VectorSet(0, w["decode_q"][0]))


def _ref_sweep(h, kind, grid, k, ivf, gp):
    L = C.CDLL(REF_LIB)
    L.ref_recall_sweep.argtypes = ([C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint64,
                                    C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_uint32,
                                    C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                    C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                    C.c_char_p, C.c_uint64])
    L.ref_last_error.restype = C.c_char_p
    K, P, D = (np.ascontiguousarray(v.data, np.float32) for v in
               (h.keys, h.prefill_queries, h.decode_queries))
    g = np.asarray(grid, np.uint32)
    buf = C.create_string_buffer(1 << 16)
    rc = L.ref_recall_sweep(K.ctypes.data, K.shape[0], K.shape[1], P.ctypes.data, P.shape[0],
                            D.ctypes.data, D.shape[0], {"flat": 0, "ivf": 1, "oodgraph": 2}[kind],
                            g.ctypes.data, len(g), k, ivf.nlist, ivf.seed, ivf.iters,
                            ivf.default_nprobe, gp.k_train, gp.max_degree, gp.ef_construction,
                            gp.edge_window, 4, buf, len(buf))
    assert rc == 0, L.ref_last_error()
    csv, jl = buf.raw.split(b"\0")[:2]
    return csv.decode(), jl.decode()


@pytest.mark.parametrize("kind,grid", [("flat", []), ("ivf", [1, 4, 16, 55]),
                                       ("oodgraph", [20, 32, 64, 128])])
def test_recall_sweep_reports_identical(head, kind, grid):
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.diagnostics import SweepParams, recall_sweep
    ivf = ra.IVFBuildParams(0, 5, 20, 8)
    gp = ra.OODGraphBuildParams(16, 12, 48, 8)
    rep = recall_sweep(head, SweepParams(kind, grid, 20, ivf, gp))
    csv, jl = _ref_sweep(head, kind, grid, 20, ivf, gp)
    assert rep.to_csv() == csv
    assert rep.to_jsonl() == jl
    assert len(rep.rows) == max(1, len(grid))


def test_recall_sweep_errors(head):
    from paper_2409_10516_b200.diagnostics import SweepParams, recall_at_k, recall_sweep
    with pytest.raises(ValueError, match="^empty parameter grid$"):
        recall_sweep(head, SweepParams("ivf", []))
    with pytest.raises(ValueError, match="^grid values must be >= 1$"):
        recall_sweep(head, SweepParams("oodgraph", [0, 128]))
    with pytest.raises(ValueError, match="^k out of range$"):
        recall_sweep(head, SweepParams("flat", [], 0))
    with pytest.raises(ValueError, match="^unknown index kind: hnsw$"):
        recall_sweep(head, SweepParams("hnsw", [8]))
    with pytest.raises(ValueError, match="^empty truth$"):
        recall_at_k([1, 2], [])
    assert recall_at_k([3, 3, 9], [3, 4]) == 1.0  # duplicates count (reference loop)
