"""The reference's OWN unit suites against the GPU backend.

oracle/Makefile `gpu-conformance` links /root/reference/proj/tests/
test_index_oodgraph.cpp, test_engine.cpp and test_attention.cpp (unmodified)
with every reference source EXCEPT src/index_oodgraph.cpp, src/attention.cpp
and src/engine.cpp, which are replaced by the drop-in TUs
paper_2409_10516_b200/host/attnindex_{oodgraph,attention,engine}_gpu.cpp over
libra_b200.so — i.e. exactly what a maintainer adopting the backend would
build. Every OODGraph build and search, every partial attention / merge and
every OODGraph decode_step in those suites then runs on the B200.

The same drop-in library (libattnindex_dropin.so) also serves the
reference's setup + decode_step through its own API, compared here with the
unmodified reference on identical inputs.
"""
import numpy as np
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("suite", ["test_index_oodgraph", "test_engine", "test_attention"])
def test_reference_suite_passes_on_gpu_backend(suite):
    exe = os.path.join(REF_DIR, "gpu_" + suite)
    if not os.path.exists(exe):
        pytest.skip("conformance binary not built (needs /root/reference at build time)")
    r = subprocess.run([exe], cwd=REF_DIR, capture_output=True, text=True, timeout=900)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed" in r.stdout


def test_reference_api_decode_through_dropin_matches_reference():
    """generate_workload + engine_init + decode_step through the reference's
    API: GPU drop-in library vs the unmodified reference, same inputs (16K,
    8 heads / 2 groups, README graph parameters): identical graphs, retrieved
    ids and scanned, outputs within 1e-12 relative."""
    from oracle.ffi import BuildParams, Oracle, available
    if not (available("ref") and available("dropin")):
        pytest.skip("reference / drop-in libraries not built")
    bp = BuildParams(128, 24, 256, 8)
    args = dict(n_ctx=16384, n_heads=8, n_kv_groups=2, seed=7, n_decode=4, params=bp,
                n_threads=8)
    ref, dq, _, _, _, _ = Oracle("ref").engine_from_workload(**args, build_workers=4)
    gpu, dq2, _, _, _, _ = Oracle("dropin").engine_from_workload(**args)
    assert np.array_equal(dq, dq2)
    for h in range(8):
        assert ref.graph_blob(h) == gpu.graph_blob(h), f"graph of head {h}"
    for s in range(4):
        q = np.ascontiguousarray(dq[:, s, :])
        ro, rom, rsc = ref.step(q, s)
        go, gom, gsc = gpu.step(q, s)
        assert np.array_equal(rom, gom) and np.array_equal(rsc, gsc), f"step {s}"
        rel = np.linalg.norm(go - ro, axis=1) / np.linalg.norm(ro, axis=1)
        assert rel.max() <= 1e-12, rel.max()
