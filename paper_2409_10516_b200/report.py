"""The `build` command's per-head index report (reference tools/main.cpp:401-480,
`cmd_build`) on top of the GPU builders, plus its `--verify` log
(main.cpp:308-321).

build_run builds every head's index on the device (flat / ivf / oodgraph,
as build_index does at main.cpp:360-374), writes each graph's OODG v1
artifact and `build_report.json` into out_dir, and returns the report path.
The report holds no timings, so it is byte-identical to the reference's for
the same workload (graphs, IVF lists and memory_bytes are exact);
tests/test_report_gpu.py checks it against oracle/_ref's restatement.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from .api import (InvalidArgument, IVFBuildParams, KVGroup, OODGraph, OODGraphBuildParams,
                  _check, flat_build, ivf_build, lib, ood_build)

KINDS = ("flat", "ivf", "oodgraph")  # index_kind_name (engine.cpp)


@dataclass
class VerifyLog:
    """main.cpp:308-321: counts checks when enabled, keeps failure texts."""

    enabled: bool = False
    checks: int = 0
    failures: List[str] = field(default_factory=list)

    def check(self, ok: bool, what: str) -> None:
        if not self.enabled:
            return
        self.checks += 1
        if not ok:
            self.failures.append(what)


def graph_csr(g: OODGraph):
    """(offsets u64[n+1], adjacency u32[E]) host copies of the graph's CSR."""
    n = g.size()
    off = np.empty(n + 1, np.uint64)
    _check(lib.ra_graph_csr(g.h, off.ctypes.data_as(_capi.c_u64p), None))
    adj = np.empty(int(off[-1]), np.uint32)
    _check(lib.ra_graph_csr(g.h, off.ctypes.data_as(_capi.c_u64p),
                            adj.ctypes.data_as(_capi.c_u32p)))
    return off, adj


def build_run(heads: Sequence, kind: str, out_dir, graph: OODGraphBuildParams = None,
              ivf: IVFBuildParams = None, seed: int = 0,
              verify: Optional[VerifyLog] = None) -> str:
    """cmd_build (main.cpp:401-480). `heads`: kvd1.HeadWorkload list (heads of
    one group share their keys/values objects, as load_workloads returns
    them). `seed` is the engine seed the IVF build takes (main.cpp:366)."""
    if kind not in KINDS:
        raise InvalidArgument("unknown index kind: " + str(kind))
    if not heads:
        raise RuntimeError("workload has no heads")
    graph = graph or OODGraphBuildParams()
    ivf = ivf or IVFBuildParams()
    v = verify or VerifyLog()
    os.makedirs(out_dir, exist_ok=True)
    arr = lambda x: np.asarray(getattr(x, "data", x), np.float32)
    kvs = {}  # one device KV group per keys object (GQA sharing)
    per_head, counted = [], set()
    kv_bytes = index_bytes = 0
    for h in heads:
        key = id(h.keys)
        if key not in kvs:
            kvs[key] = KVGroup(arr(h.keys))
        kv = kvs[key]
        if kind == "flat":
            idx = flat_build(kv)
        elif kind == "ivf":
            idx = ivf_build(kv, IVFBuildParams(ivf.nlist, seed, ivf.iters, ivf.default_nprobe))
        else:
            idx = ood_build(kv, arr(h.prefill_queries), graph)
        entry = {"head": int(h.head_id), "kv_group": int(h.kv_group_id)}
        if kind == "oodgraph":
            name = f"head{h.head_id}.oodg"
            path = os.path.join(out_dir, name)
            blob = idx.serialize()
            with open(path, "wb") as f:
                f.write(blob)
            entry["artifact"] = name
            off, _ = graph_csr(idx)
            deg = np.diff(off.astype(np.int64))
            entry["edges"] = int(deg.sum())
            entry["degree_histogram"] = [
                int(c) for c in np.bincount(deg, minlength=idx.max_degree_bound() + 1)]
            entry["entry_point"] = idx.entry_point()
            v.check(idx.reachable_count() == idx.size(),
                    f"build: head {h.head_id} fully reachable")
            back = OODGraph.load(kv, path)
            v.check(back.serialize() == blob, f"build: head {h.head_id} artifact round-trip")
        elif kind == "ivf":
            entry["artifact"] = None
            entry["nlist"] = idx.nlist()
            _, off, ids = idx.export()
            n = idx.size()
            ok = bool(((ids < n).all() and np.unique(ids).size == ids.size)) if ids.size else True
            v.check(ok and int(off[-1]) == n, f"build: head {h.head_id} ivf lists partition keys")
        else:
            entry["artifact"] = None
            entry["note"] = "no preprocessing"
        entry["memory_bytes"] = idx.memory_bytes()
        index_bytes += idx.memory_bytes()
        for vs in (h.keys, h.values):
            if id(vs) not in counted:
                counted.add(id(vs))
                kv_bytes += arr(vs).size * 4
        per_head.append(entry)
    keys0 = arr(heads[0].keys)
    report = {"kind": kind, "n_heads": len(heads), "n_keys": int(keys0.shape[0]),
              "heads": per_head, "kv_bytes": int(kv_bytes), "index_bytes": int(index_bytes)}
    out = os.path.join(out_dir, "build_report.json")
    with open(out, "w") as f:
        # nlohmann::json dump(2): object keys sorted, 2-space indent
        f.write(json.dumps(report, indent=2, sort_keys=True, ensure_ascii=False) + "\n")
    return out
