"""Host-side report formatting (CPU only): recall_at_k semantics
(diagnostics.cpp:132-141), SweepReport::to_csv / to_jsonl text
(diagnostics.cpp:196-225) and the build command's VerifyLog
(tools/main.cpp:308-321). The GPU suites compare whole reports with the
reference's; these pin the formatting rules themselves."""
import json

import pytest


def _diag():
    from paper_2409_10516_b200 import diagnostics
    return diagnostics


def test_recall_at_k():
    d = _diag()
    assert d.recall_at_k([1, 2, 3], [3, 2, 1, 0]) == 0.75
    assert d.recall_at_k([], [5]) == 0.0
    assert d.recall_at_k([7, 7], [7, 8]) == 1.0  # each retrieved occurrence counts
    with pytest.raises(ValueError, match="^empty truth$"):
        d.recall_at_k([1], [])


def test_sweep_report_text():
    d = _diag()
    rep = d.SweepReport([d.SweepRow("oodgraph", 128, 0.95, 0.0251234567891, 24),
                         d.SweepRow("flat", 0, 1.0, 1.0, 24),
                         d.SweepRow("ivf", 8, 1 / 3, 2e-5, 3)])
    assert rep.to_csv() == ("index_kind,param,recall_at_k,scan_fraction,n_queries\n"
                            "oodgraph,128,0.95,0.02512345679,24\n"
                            "flat,0,1,1,24\n"
                            "ivf,8,0.3333333333,2e-05,3\n")
    lines = rep.to_jsonl().splitlines()
    assert lines[0] == ('{"index_kind":"oodgraph","param":128,"recall_at_k":0.95,'
                        '"scan_fraction":0.0251234567891,"n_queries":24}')
    assert json.loads(lines[2])["recall_at_k"] == 1 / 3
    assert list(json.loads(lines[1])) == ["index_kind", "param", "recall_at_k",
                                          "scan_fraction", "n_queries"]


def test_verify_log():
    from paper_2409_10516_b200.report import VerifyLog
    off = VerifyLog()
    off.check(False, "ignored")
    assert off.checks == 0 and off.failures == []
    v = VerifyLog(enabled=True)
    v.check(True, "a")
    v.check(False, "build: head 3 fully reachable")
    assert v.checks == 2 and v.failures == ["build: head 3 fully reachable"]
