"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, host-only entry points behave like the reference, and with
no GPU every device entry point fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, has_gpu


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ra_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ra_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2409_10516_b200 as ra
    syms = header_symbols()
    assert len(syms) >= 30
    lib = C.CDLL(ra._capi._build.LIB)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares every one of them
    assert sorted(ra.EXPORTED) == syms


def test_library_is_sm100a_only():
    import subprocess
    import paper_2409_10516_b200 as ra
    out = subprocess.run(["cuobjdump", "--list-elf", ra._capi._build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_static_partition_matches_reference_formula():
    # test_attention.cpp:198-236
    import paper_2409_10516_b200 as ra
    p = ra.static_partition(100000, 128, 512)
    assert len(p.static_set) == 640 and len(p.dynamic_pool) == 100000 - 640
    assert p.static_set[127] == 127 and p.static_set[128] == 100000 - 512
    p = ra.static_partition(500, 128, 512)
    assert len(p.static_set) == 500 and len(p.dynamic_pool) == 0
    p = ra.static_partition(1000, 128, 512)
    assert p.static_set[128] == 488 and p.dynamic_pool[0] == 128 and p.dynamic_pool[-1] == 487
    for t in (0, 1, 100, 640, 641, 5000):
        p = ra.static_partition(t, 128, 512)
        allids = np.sort(np.concatenate([p.static_set, p.dynamic_pool]))
        np.testing.assert_array_equal(allids, np.arange(t))
    with pytest.raises(ra.InvalidArgument, match="context length exceeds id width"):
        ra.static_partition(1 << 33, 128, 512)


def test_static_partition_matches_oracle(port):
    import paper_2409_10516_b200 as ra
    for t, si, sl in [(2048, 128, 512), (700, 16, 64), (10, 0, 0), (5, 8, 8)]:
        p = ra.static_partition(t, si, sl)
        w, pool = port.static_partition(t, si, sl)
        np.testing.assert_array_equal(p.static_set, w)
        np.testing.assert_array_equal(p.dynamic_pool, pool)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    import paper_2409_10516_b200 as ra
    h = C.c_void_p()
    rc = ra.lib.ra_ctx_create(0, C.byref(h))
    assert rc == 3  # RA_ERR_CUDA
    assert b"no CUDA device" in ra.lib.ra_last_error()
