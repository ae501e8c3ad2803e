"""The fused decode step (search kernel + W / Omega partials + merge in one
launch) and the three-kernel path it replaces: which one an engine runs, and
that the three-kernel path still matches the reference (it serves bf16
groups and throughput-mode batches, and RA_FUSED_ATTN=0)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.ffi import available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("port"), reason="oracle not built")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _engine(dtype):
    import paper_2409_10516_b200 as ra
    from oracle.ffi import Oracle
    w = Oracle("port").generate_workload(4000, 64, 32, 4, 1, seed=7, n_decode=4)
    kv = ra.KVGroup(w["keys"][0], w["values"][0], dtype=dtype)
    gs = [ra.ood_build(kv, w["prefill_q"][h], ra.OODGraphBuildParams(16, 12, 48, 8))
          for h in range(4)]
    return ra.Engine([kv], gs, ra.EngineConfig(16, 64, 20, 32)), w


def test_kernels_per_step():
    if os.environ.get("RA_FUSED_ATTN") == "0":
        pytest.skip("fusion disabled in this process")
    eng, _ = _engine("f32")
    assert eng.kernels_per_step() == 1
    eng16, _ = _engine("bf16_attn")
    assert eng16.kernels_per_step() == 3
    engb, _ = _engine("bf16")  # full bf16: the tail reads the f32 copy (same rounded values)
    assert engb.kernels_per_step() == 1


def test_fused_and_three_kernel_steps_agree(tmp_path):
    """Same step with fusion on (this process) and off (a child process):
    identical Omega ids and scanned, outputs within 1e-13 relative (the W
    partials are chunked differently: 24-row vs 64-row chunks)."""
    eng, w = _engine("f32")
    Q = np.stack([w["decode_q"][h][0] for h in range(4)])
    out, om, sc = eng.decode_step(Q)
    np.save(tmp_path / "q.npy", Q)
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
from test_fused_gpu import _engine
eng, w = _engine("f32")
assert eng.kernels_per_step() == 3
out, om, sc = eng.decode_step(np.load({str(tmp_path / 'q.npy')!r}))
np.savez({str(tmp_path / 'r.npz')!r}, out=out, om=om, sc=sc)
"""
    env = dict(os.environ, RA_FUSED_ATTN="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    ref = np.load(tmp_path / "r.npz")
    np.testing.assert_array_equal(om, ref["om"])
    np.testing.assert_array_equal(sc, ref["sc"])
    rel = np.abs(out - ref["out"]).max() / np.abs(ref["out"]).max()
    assert rel <= 1e-13, rel


def test_three_kernel_path_matches_reference():
    """The engine-vs-reference decode_step suite with fusion disabled."""
    env = dict(os.environ, RA_FUSED_ATTN="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_attention_gpu.py"), "-k",
                        "engine_matches or window"], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:]


@pytest.mark.parametrize("M,d", [(2, 32), (4, 32), (8, 16), (6, 64)])
def test_fused_step_small_degree_matches_oracle(M, d):
    """Low-degree graphs give the helpers short tiles; the fused tail still
    stages its W partials and V rows there (the launch grows the tiles), and
    the step equals the reference's run_head (engine.cpp:69-101)."""
    import paper_2409_10516_b200 as ra
    from oracle.ffi import BuildParams, Oracle
    port = Oracle("port")
    w = port.generate_workload(1500, 64, d, 2, 1, seed=3, n_decode=2)
    bp = BuildParams(k_train=8, max_degree=M, ef_construction=16)
    blobs = [port.graph_build(w["keys"][0], w["prefill_q"][h], bp) for h in range(2)]
    kv = ra.KVGroup(w["keys"][0], w["values"][0])
    eng = ra.Engine([kv], [ra.OODGraph.from_blob(kv, b) for b in blobs],
                    ra.EngineConfig(16, 64, 20, 32))
    if os.environ.get("RA_FUSED_ATTN") != "0" and d >= 32:
        assert eng.kernels_per_step() == 1
    Q = np.ascontiguousarray(w["decode_q"][:, 0, :])
    out, om, sc = eng.decode_step(Q)
    W = ra.static_partition(1500, 16, 64).static_set
    for h in range(2):
        r = port.graph(w["keys"][0], blobs[h]).search(Q[h], 20, W, 32)
        assert np.array_equal(om[h][: len(r.ids)], r.ids) and int(sc[h]) == r.scanned
        pw = port.partial_attention(Q[h], w["keys"][0], w["values"][0], W)
        po = port.partial_attention(Q[h], w["keys"][0], w["values"][0], r.ids)
        ref = port.merge(pw, po, d)[0]
        # W partials are summed per chunk and merged (the reference sums W in
        # one pass): a few ulp, far inside north_star's 1e-3
        assert np.linalg.norm(out[h] - ref) / np.linalg.norm(ref) <= 1e-9
