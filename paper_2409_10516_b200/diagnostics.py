"""recall_sweep and its reports (reference diagnostics.cpp:132-225 /
diagnostics.hpp:43-71) over the GPU indexes: the flat ground truth, the IVF
and graph searches all run batched on the device; the reductions follow the
reference's order so the CSV / JSONL reports are byte-identical to its
(the searches return the reference's exact ids and `scanned`).
tests/test_diagnostics_gpu.py checks them against oracle/_ref's restatement.
"""
from __future__ import annotations

import bisect
import json
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .api import (InvalidArgument, IVFBuildParams, OODGraphBuildParams, flat_build, ivf_build,
                  ood_build, search_batch, KVGroup)


def recall_at_k(retrieved, truth) -> float:
    """diagnostics.cpp:132-141: |retrieved ∩ truth| / |truth| (retrieved
    duplicates count each time, as the reference's loop does)."""
    if len(truth) == 0:
        raise InvalidArgument("empty truth")
    s = sorted(int(t) for t in truth)
    hits = 0
    for i in retrieved:
        j = bisect.bisect_left(s, int(i))
        hits += j < len(s) and s[j] == int(i)
    return hits / len(truth)


@dataclass
class SweepParams:
    """diagnostics.hpp:58-65"""

    index_kind: str = "oodgraph"  # "flat" | "ivf" | "oodgraph"
    grid: List[int] = field(default_factory=list)
    k: int = 100
    ivf: IVFBuildParams = field(default_factory=IVFBuildParams)
    graph: OODGraphBuildParams = field(default_factory=OODGraphBuildParams)
    n_threads: int = 1  # accepted for parity; the device does the parallel part


@dataclass
class SweepRow:
    index_kind: str
    param: int
    recall_at_k: float
    scan_fraction: float
    n_queries: int


def _fmt(v: float) -> str:  # fmt_double (diagnostics.cpp:43-47)
    return "%.10g" % v


@dataclass
class SweepReport:
    rows: List[SweepRow] = field(default_factory=list)

    def to_csv(self) -> str:
        """SweepReport::to_csv (diagnostics.cpp:196-211)"""
        out = "index_kind,param,recall_at_k,scan_fraction,n_queries\n"
        for r in self.rows:
            out += (f"{r.index_kind},{r.param},{_fmt(r.recall_at_k)},{_fmt(r.scan_fraction)},"
                    f"{r.n_queries}\n")
        return out

    def to_jsonl(self) -> str:
        """SweepReport::to_jsonl (diagnostics.cpp:213-225): ordered_json dump()."""
        return "".join(json.dumps({"index_kind": r.index_kind, "param": r.param,
                                   "recall_at_k": r.recall_at_k,
                                   "scan_fraction": r.scan_fraction,
                                   "n_queries": r.n_queries}, separators=(",", ":"),
                                  ensure_ascii=False) + "\n" for r in self.rows)


def _seqmean(xs) -> float:
    s = 0.0
    for x in xs:  # std::accumulate order
        s += x
    return s / len(xs)


def recall_sweep(head, p: SweepParams = None) -> SweepReport:
    """recall_sweep (diagnostics.cpp:143-194). `head`: a kvd1.HeadWorkload
    (or anything with keys / prefill_queries / decode_queries)."""
    p = p or SweepParams()
    arr = lambda v: np.ascontiguousarray(getattr(v, "data", v), np.float32)
    keys, dq = arr(head.keys), arr(head.decode_queries)
    n, nq = keys.shape[0], dq.shape[0]
    if nq == 0:
        raise InvalidArgument("no decode queries")
    if p.k < 1 or p.k > n:
        raise InvalidArgument("k out of range")
    kv = KVGroup(keys)
    flat = flat_build(kv)
    truth = [r.ids for r in flat.search_batch(dq, p.k)]
    rep = SweepReport()

    def add_row(kind, param, results):
        rec = [recall_at_k(r.ids, truth[i]) for i, r in enumerate(results)]
        scan = [r.scanned / n for r in results]
        rep.rows.append(SweepRow(kind, int(param), _seqmean(rec), _seqmean(scan), nq))

    if p.index_kind == "flat":
        add_row("flat", 0, flat.search_batch(dq, p.k))
        return rep
    if not p.grid:
        raise InvalidArgument("empty parameter grid")
    if any(g < 1 for g in p.grid):
        raise InvalidArgument("grid values must be >= 1")
    if p.index_kind == "ivf":
        idx = ivf_build(kv, p.ivf)
        for g in p.grid:
            add_row("ivf", g, idx.search_batch(dq, p.k, None, g))
    elif p.index_kind == "oodgraph":
        g0 = ood_build(kv, arr(head.prefill_queries), p.graph)
        for g in p.grid:
            add_row("oodgraph", g, search_batch([g0], dq, p.k, None, g).host())
    else:
        raise InvalidArgument("unknown index kind: " + p.index_kind)
    return rep
