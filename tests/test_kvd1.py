"""KVD1 files + manifest (io.hpp / io.cpp) against the reference's own
writer (oracle/_ref save_workloads): byte-identical files, round trip, and
the reference's load errors. CPU only."""
import ctypes as C
import filecmp
import os
import struct

import numpy as np
import pytest

from oracle.ffi import REF_LIB, Oracle, available


def _kvd1():
    from paper_2409_10516_b200 import kvd1
    return kvd1


@pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
def test_save_workloads_byte_identical_to_reference(tmp_path):
    kvd1 = _kvd1()
    n_ctx, d_model, d_head, H, G, seed, n_dec = 300, 64, 32, 4, 2, 7, 5
    lib = C.CDLL(REF_LIB)
    lib.ref_save_workloads.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint64, C.c_uint64, C.c_char_p]
    ref_dir = tmp_path / "ref"
    assert lib.ref_save_workloads(n_ctx, d_model, d_head, H, G, seed, n_dec,
                                  str(ref_dir).encode()) == 0
    w = Oracle("ref").generate_workload(n_ctx, d_model, d_head, H, G, seed=seed, n_decode=n_dec)
    hpg = H // G
    keys = [kvd1.VectorSet(1, w["keys"][g]) for g in range(G)]
    vals = [kvd1.VectorSet(2, w["values"][g]) for g in range(G)]
    heads = [kvd1.HeadWorkload(h, h // hpg, kvd1.VectorSet(0, w["prefill_q"][h]),
                               keys[h // hpg], vals[h // hpg],
                               kvd1.VectorSet(0, w["decode_q"][h])) for h in range(H)]
    ours = tmp_path / "ours"
    kvd1.save_workloads(heads, G, ours)
    names = sorted(os.listdir(ref_dir))
    assert names == sorted(os.listdir(ours))
    for nm in names:
        assert filecmp.cmp(ref_dir / nm, ours / nm, shallow=False), nm
    # load back: shared group storage, identical arrays
    back = kvd1.load_workloads(ours / "manifest.json")
    assert back[0].keys is back[1].keys and back[0].keys is not back[2].keys
    for h in range(H):
        np.testing.assert_array_equal(back[h].prefill_queries.data, w["prefill_q"][h])
        np.testing.assert_array_equal(back[h].values.data, w["values"][h // hpg])
        assert back[h].kv_group_id == h // hpg


def test_load_vectors_errors(tmp_path):
    kvd1 = _kvd1()
    good = b"KVD1" + struct.pack("<IB3xQI4x", 1, 1, 2, 3) + np.arange(6, dtype="<f4").tobytes()
    p = tmp_path / "x.kvd"

    def expect(blob, what):
        p.write_bytes(blob)
        with pytest.raises(Exception, match="^kvd1 format error in .*: " + what + "$"):
            kvd1.load_vectors(p)
    p.write_bytes(good)
    vs = kvd1.load_vectors(p)
    assert vs.role == 1 and vs.data.shape == (2, 3)
    expect(good[:10], "truncated header")
    expect(b"KVD2" + good[4:], "bad magic")
    expect(good[:4] + struct.pack("<I", 2) + good[8:], "unsupported version 2")
    expect(good[:8] + bytes([3]) + good[9:], "bad role 3")
    expect(good[:20] + struct.pack("<I", 0) + good[24:], "d must be >= 1")
    expect(good[:-4], "truncated payload")
    expect(good + b"\0", "trailing bytes after payload")
    if available("ref"):  # the same texts from the reference itself
        lib = C.CDLL(REF_LIB)
        lib.ref_load_vectors_check.argtypes = [C.c_char_p]
        lib.ref_last_error.restype = C.c_char_p
        p.write_bytes(good + b"\0")
        assert lib.ref_load_vectors_check(str(p).encode()) != 0
        assert lib.ref_last_error().decode().endswith("trailing bytes after payload")
