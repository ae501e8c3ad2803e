"""`build` report (tools/main.cpp:401-480) on the GPU builders vs the
reference's own builders (oracle/_ref ref_build_report, a restatement of
cmd_build over the unmodified library) on the same KVD1 workload:
every OODG artifact byte-identical, the same report object and verify
checks all passing, for flat / ivf / oodgraph.

The report text is compared as stock nlohmann::json dump(2) output (the
reference vendors nlohmann under vendor/, absent here). The copy the oracle
compiles against (cudnn_frontend's thirdparty/nlohmann/json.hpp:20609-20613)
carries a local patch that prints integer arrays on one line, so its bytes
differ from stock in the degree histogram only; the parsed objects must be
equal and our bytes must be stock dump(2) of that object."""
import ctypes as C
import filecmp
import json
import os

import pytest

from oracle.ffi import REF_LIB, available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")]

KIND_ID = {"flat": 0, "ivf": 1, "oodgraph": 2}


def _ref():
    L = C.CDLL(REF_LIB)
    L.ref_save_workloads.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint32, C.c_uint64, C.c_uint64, C.c_char_p]
    L.ref_build_report.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint32, C.c_uint32,
                                   C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                   C.c_uint32, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64)]
    L.ref_last_error.restype = C.c_char_p
    return L


@pytest.fixture(scope="module")
def workload(tmp_path_factory):
    d = tmp_path_factory.mktemp("wl")
    L = _ref()
    # 4 heads over 2 KV groups, 1500 keys, d_head 32 (acceptance-style generator)
    assert L.ref_save_workloads(1500, 64, 32, 4, 2, 7, 3, str(d).encode()) == 0
    return d


@pytest.mark.parametrize("kind", ["oodgraph", "ivf", "flat"])
def test_build_report_byte_identical(workload, tmp_path, kind):
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200 import kvd1
    from paper_2409_10516_b200.report import VerifyLog, build_run
    L = _ref()
    gp = ra.OODGraphBuildParams(16, 12, 48, 8)
    ivf = ra.IVFBuildParams(0, 0, 20, 8)
    seed = 3
    ref_dir = tmp_path / "ref"
    checks, fails = C.c_uint64(), C.c_uint64()
    rc = L.ref_build_report(str(workload / "manifest.json").encode(), str(ref_dir).encode(),
                            KIND_ID[kind], gp.k_train, gp.max_degree, gp.ef_construction,
                            gp.edge_window, ivf.nlist, seed, ivf.iters, ivf.default_nprobe, 4, 1,
                            C.byref(checks), C.byref(fails))
    assert rc == 0, L.ref_last_error()
    heads = kvd1.load_workloads(workload / "manifest.json")
    v = VerifyLog(enabled=True)
    out = build_run(heads, kind, tmp_path / "ours", gp, ivf, seed=seed, verify=v)
    assert os.path.basename(out) == "build_report.json"
    assert v.failures == [] and fails.value == 0
    assert v.checks == checks.value
    names = sorted(os.listdir(ref_dir))
    assert names == sorted(os.listdir(tmp_path / "ours"))
    for nm in names:
        if nm == "build_report.json":
            ours = (tmp_path / "ours" / nm).read_text()
            obj = json.loads((ref_dir / nm).read_text())
            assert json.loads(ours) == obj
            assert ours == json.dumps(obj, indent=2, sort_keys=True, ensure_ascii=False) + "\n"
            continue
        assert filecmp.cmp(ref_dir / nm, tmp_path / "ours" / nm, shallow=False), nm


def test_build_report_errors(tmp_path):
    from paper_2409_10516_b200.report import build_run
    with pytest.raises(ValueError, match="unknown index kind"):
        build_run([object()], "hnsw", tmp_path)
    with pytest.raises(RuntimeError, match="workload has no heads"):
        build_run([], "flat", tmp_path)
