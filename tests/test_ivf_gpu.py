"""GPU IVF (index_ivf.cpp) vs the reference itself (oracle/_ref, Eigen
restated in index order): centroids, lists and search results identical;
the reference's errors; scan contrast vs the graph (acceptance C6 shape)."""
import ctypes as C

import numpy as np
import pytest

from oracle.ffi import REF_LIB, available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")]


class RefIVF:
    def __init__(self, keys, nlist, seed, iters, nprobe):
        self.lib = C.CDLL(REF_LIB)
        L = self.lib
        L.ref_ivf_build.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64,
                                    C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]
        L.ref_ivf_nlist.restype = C.c_uint32
        L.ref_ivf_nlist.argtypes = [C.c_void_p]
        L.ref_ivf_export.argtypes = [C.c_void_p] * 4
        L.ref_ivf_search.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p,
                                     C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p]
        L.ref_ivf_free.argtypes = [C.c_void_p]
        self.keys = np.ascontiguousarray(keys, np.float32)
        self.h = C.c_void_p()
        assert L.ref_ivf_build(self.keys.ctypes.data, self.keys.shape[0], self.keys.shape[1],
                               nlist, seed, iters, nprobe, C.byref(self.h)) == 0
        self.nlist = L.ref_ivf_nlist(self.h)

    def export(self):
        n, d = self.keys.shape
        cent = np.empty((self.nlist, d), np.float32)
        off = np.empty(self.nlist + 1, np.uint32)
        ids = np.empty(n, np.uint32)
        assert self.lib.ref_ivf_export(self.h, cent.ctypes.data, off.ctypes.data,
                                       ids.ctypes.data) == 0
        return cent, off, ids

    def search(self, q, k, mask=None, nprobe=-1):
        q = np.ascontiguousarray(q, np.float32)
        m = np.ascontiguousarray(mask if mask is not None else np.zeros(0), np.uint32)
        ids = np.zeros(k, np.uint32)
        sc = np.zeros(k, np.float32)
        n_out, scanned, tr = C.c_uint64(), C.c_uint64(), C.c_uint8()
        assert self.lib.ref_ivf_search(self.h, q.ctypes.data, q.size, k, m.ctypes.data, m.size,
                                       nprobe, ids.ctypes.data, sc.ctypes.data, C.byref(n_out),
                                       C.byref(scanned), C.byref(tr)) == 0
        return ids[: n_out.value], sc[: n_out.value], scanned.value, bool(tr.value)

    def __del__(self):
        self.lib.ref_ivf_free(self.h)


@pytest.mark.parametrize("n,d,nlist,iters", [(3000, 32, 0, 20), (5000, 64, 40, 8),
                                             (600, 16, 600, 3), (800, 128, 1, 2)])
def test_ivf_build_and_search_match_reference(port, n, d, nlist, iters):
    import paper_2409_10516_b200 as ra
    w = port.generate_workload(n, 256, d, 1, 1, seed=n + d, n_decode=12)
    K = w["keys"][0]
    ref = RefIVF(K, nlist, 5, iters, 8)
    ix = ra.IVFIndex(ra.KVGroup(K), ra.IVFBuildParams(nlist, 5, iters, 8))
    assert ix.nlist() == ref.nlist
    rc, ro, ri = ref.export()
    gc, go, gi = ix.export()
    np.testing.assert_array_equal(go, ro)
    np.testing.assert_array_equal(gi, ri)
    np.testing.assert_array_equal(gc, rc)
    Q = w["decode_q"][0]
    mask = np.sort(np.random.default_rng(1).choice(n, size=n // 10, replace=False)).astype(np.uint32)
    for m in (None, mask):
        for k, nprobe in ((10, None), (100, min(3, ix.nlist())), (n // 2, ix.nlist())):
            res = ix.search_batch(Q, k, m, nprobe)
            for qi in range(len(Q)):
                ids, sc, scanned, tr = ref.search(Q[qi], k, m, -1 if nprobe is None else nprobe)
                np.testing.assert_array_equal(res[qi].ids, ids)
                np.testing.assert_array_equal(res[qi].scores, sc)
                assert res[qi].scanned == scanned and res[qi].truncated == tr


def test_ivf_errors():
    import paper_2409_10516_b200 as ra
    K = np.random.default_rng(2).standard_normal((50, 8)).astype(np.float32)
    with pytest.raises(ra.InvalidArgument, match="^nlist out of range$"):
        ra.IVFIndex(ra.KVGroup(K), ra.IVFBuildParams(nlist=51))
    ix = ra.IVFIndex(ra.KVGroup(K), ra.IVFBuildParams(nlist=5))
    q = np.ones(8, np.float32)
    with pytest.raises(ra.InvalidArgument, match="^nprobe out of range$"):
        ix.search(q, 3, None, 6)
    with pytest.raises(ra.InvalidArgument, match="^k out of range$"):
        ix.search(q, 0)
    with pytest.raises(ra.InvalidArgument, match="^query dimension mismatch$"):
        ix.search(np.ones(7, np.float32), 1)
    assert ix.kind() == "ivf" and ix.memory_bytes() == 5 * 8 * 4 + 50 * 4
