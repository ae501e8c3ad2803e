"""decode_run, its trace and summary, full attention and the memory report
(reference engine.hpp:45-136 / engine.cpp:117-194, attention.cpp:38-60,159-168)
on top of the GPU Engine.

The trace is produced in the reference's (step, head) order and formats;
without `compute_reference` the JSONL is byte-identical to the reference's
`DecodeTrace::to_jsonl` (ids and `scanned` are exact). With it, each entry's
mse uses the GPU full attention (device exp, <= 1 ulp per term), so mse
agrees with the reference to ~1e-12 relative rather than bit-for-bit.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import _capi
from .api import Engine, InvalidArgument, KVGroup, _check, _dev, _ptr, lib


@dataclass
class TraceEntry:
    """engine.hpp:57-65"""

    step: int
    head: int
    omega: np.ndarray
    scanned: int
    w_size: int
    out: np.ndarray
    mse: Optional[float] = None


@dataclass
class DecodeTrace:
    entries: List[TraceEntry] = field(default_factory=list)

    def to_jsonl(self, include_omega: bool) -> str:
        """DecodeTrace::to_jsonl (engine.cpp:157-170): one compact object per
        (step, head), keys in insertion order."""
        out = []
        for e in self.entries:
            j = {"step": e.step, "head": e.head}
            if include_omega:
                j["omega_ids"] = [int(x) for x in e.omega]
            j["scanned"] = e.scanned
            if e.mse is not None:
                j["mse"] = e.mse
            out.append(json.dumps(j, separators=(",", ":")) + "\n")
        return "".join(out)


@dataclass
class DecodeSummary:
    """engine.hpp:73-86"""

    n_steps: int = 0
    n_heads: int = 0
    mean_scan_fraction: float = 0.0
    mean_scanned: float = 0.0
    total_scanned: int = 0
    mean_mse: float = 0.0
    max_mse: float = 0.0

    def to_json(self) -> str:
        """DecodeSummary::to_json (engine.cpp:172-182): dump(2), insertion order."""
        return json.dumps({"n_steps": self.n_steps, "n_heads": self.n_heads,
                           "mean_scan_fraction": float(self.mean_scan_fraction),
                           "mean_scanned": float(self.mean_scanned),
                           "total_scanned": self.total_scanned,
                           "mean_mse": float(self.mean_mse), "max_mse": float(self.max_mse)},
                          indent=2)


@dataclass
class DecodeResult:
    trace: DecodeTrace
    summary: DecodeSummary


def full_attention(q, kv: KVGroup) -> np.ndarray:
    """full_attention (attention.cpp:38-60) on the GPU: softmax over every
    key in index order (the partial-attention kernel over all ids)."""
    q = np.asarray(q, np.float32).reshape(-1)
    if q.size != kv.d:
        raise InvalidArgument("query dimension mismatch")
    if kv.n == 0:
        raise InvalidArgument("empty context")
    ctx = kv.ctx.bind_stream()
    dev = torch.device("cuda", ctx.device)
    qd = _dev(q.reshape(1, -1), torch.float32, dev)
    ix = torch.arange(kv.n, dtype=torch.int32, device=dev)
    m = torch.tensor([kv.n], dtype=torch.int32, device=dev)
    out = torch.empty((1, kv.d), dtype=torch.float64, device=dev)
    zm = torch.empty(1, dtype=torch.float64, device=dev)
    es = torch.empty(1, dtype=torch.float64, device=dev)
    _check(lib.ra_partial_attention(ctx.h, kv.h, 1, _ptr(qd), _ptr(ix), int(kv.n), _ptr(m),
                                    _ptr(out), _ptr(zm), _ptr(es)))
    return out[0].cpu().numpy()


def mse(approx, exact) -> float:
    """attention.cpp:159-168 (in-order sum)."""
    a, b = np.asarray(approx, np.float64), np.asarray(exact, np.float64)
    if a.shape != b.shape:
        raise InvalidArgument("mse dimension mismatch")
    acc = 0.0
    for x, y in zip(a.tolist(), b.tolist()):
        acc += (x - y) * (x - y)
    return acc / float(a.size)


def decode_run(engine: Engine, decode_queries, n_steps: int,
               compute_reference: bool = False) -> DecodeResult:
    """decode_run (engine.cpp:117-155): decode_queries[h] holds head h's stored
    decode queries ([H, >= n_steps, d]); steps run in order, every head of a
    step in one GPU decode step; the summary aggregates in (step, head) order."""
    dq = np.asarray(decode_queries, np.float32)
    H = engine.H
    if dq.shape[0] != H or dq.shape[1] < n_steps:
        raise InvalidArgument("insufficient decode queries")
    res = DecodeResult(DecodeTrace(), DecodeSummary(n_steps=n_steps, n_heads=H))
    hpg = H // len(engine.groups)
    for step in range(n_steps):
        Q = np.ascontiguousarray(dq[:, step, :])
        out, omega, scanned = engine.decode_step(Q)
        for h in range(H):
            e = TraceEntry(step, h, omega[h].copy(), int(scanned[h]), engine.w_size, out[h].copy())
            if compute_reference:
                e.mse = mse(out[h], full_attention(Q[h], engine.groups[h // hpg]))
            res.trace.entries.append(e)
    s = res.summary
    with_mse = 0
    for e in res.trace.entries:
        pool = engine.t - e.w_size
        s.total_scanned += e.scanned
        s.mean_scanned += float(e.scanned)
        if pool > 0:
            s.mean_scan_fraction += float(e.scanned) / float(pool)
        if e.mse is not None:
            with_mse += 1
            s.mean_mse += e.mse
            s.max_mse = max(s.max_mse, e.mse)
    n = len(res.trace.entries)
    if n:
        s.mean_scanned /= float(n)
        s.mean_scan_fraction /= float(n)
    if with_mse:
        s.mean_mse /= float(with_mse)
    return res


def engine_memory(engine: Engine):
    """engine_memory (engine.cpp:184-194): (kv_bytes counted once per group,
    index_bytes summed over heads)."""
    kv = sum(g.n * g.d * 4 * 2 for g in engine.groups)
    idx = sum(g.memory_bytes() for g in engine.graphs)
    return kv, idx
