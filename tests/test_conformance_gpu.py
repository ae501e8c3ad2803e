"""The reference's OWN unit suites against the GPU backend.

oracle/Makefile `gpu-conformance` links /root/reference/proj/tests/
test_index_oodgraph.cpp and test_engine.cpp (unmodified) with every reference
source EXCEPT src/index_oodgraph.cpp, which is replaced by the drop-in TU
paper_2409_10516_b200/host/attnindex_oodgraph_gpu.cpp over libra_b200.so —
i.e. exactly what a maintainer adopting the backend would build. Every
OODGraph build and search in those suites then runs on the B200.
"""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("suite", ["test_index_oodgraph", "test_engine"])
def test_reference_suite_passes_on_gpu_backend(suite):
    exe = os.path.join(REF_DIR, "gpu_" + suite)
    if not os.path.exists(exe):
        pytest.skip("conformance binary not built (needs /root/reference at build time)")
    r = subprocess.run([exe], cwd=REF_DIR, capture_output=True, text=True, timeout=900)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed" in r.stdout
