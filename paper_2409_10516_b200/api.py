"""Host-side mirror of the reference's attnindex C++ API over libra_b200.so.

Names, argument meaning and error behaviour follow /root/reference/proj/include/
attnindex/{index.hpp,index_oodgraph.hpp,attention.hpp,engine.hpp}:
std::invalid_argument -> ``InvalidArgument`` (a ValueError) and
std::runtime_error -> ``GraphError`` (a RuntimeError), with the reference's
exact messages. All compute runs in the CUDA library; torch is used only to
own device buffers and streams.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi
from ._capi import lib

U32_MAX = 0xFFFFFFFF


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class GraphError(RuntimeError):
    """std::runtime_error in the reference (OODG blob / file errors)."""


class CudaError(RuntimeError):
    """CUDA failure or no sm_100a device (there is no CPU fallback)."""


def _check(rc: int) -> None:
    if rc == _capi.RA_OK:
        return
    msg = lib.ra_last_error().decode()
    if rc == _capi.RA_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == _capi.RA_ERR_RUNTIME:
        raise GraphError(msg)
    raise CudaError(msg)


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return t.ctypes.data


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------
class Context:
    """ra_ctx: device + stream + scratch. One per thread (see default_context)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        _check(lib.ra_ctx_create(device, C.byref(h)))
        self.h = h

    def bind_stream(self, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(lib.ra_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream)))
        return self

    def synchronize(self):
        _check(lib.ra_ctx_synchronize(self.h))

    def set_search_kernel(self, name: Optional[str]):
        """Graph-search kernel variant for this context ("auto", "lat",
        "tp", "tps", "tpr", "cta", "warp"; None = default). Results are
        identical across variants; engines read it at creation."""
        _check(lib.ra_ctx_set_search_kernel(self.h, None if name is None else name.encode()))

    def close(self):
        if getattr(self, "h", None):
            lib.ra_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context(device: Optional[int] = None) -> Context:
    device = torch.cuda.current_device() if device is None else device
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device].bind_stream()


def _dev(x, dtype, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device, dtype=dtype)


# ---------------------------------------------------------------------------
# KV groups  (types.hpp VectorSet / HeadWorkload sharing)
# ---------------------------------------------------------------------------
class KVGroup:
    """One GQA group's keys (and values) resident in HBM; shared by its heads
    the way HeadWorkload shares shared_ptr<const VectorSet> (types.hpp:54-61)."""

    def __init__(self, keys, values=None, ctx: Optional[Context] = None, dtype: str = "f32"):
        """dtype "bf16": K and V are rounded to bf16 (nearest even) and the
        decode path reads bf16 rows (half the HBM bytes); results equal the
        reference's on the rounded inputs (keys_tensor() holds them as f32).
        dtype "bf16_attn": the search keeps the exact f32 keys (retrieved ids
        identical to f32) and only the sparse attention reads bf16 K/V."""
        if dtype not in ("f32", "bf16", "bf16_attn"):
            raise InvalidArgument("dtype must be f32, bf16 or bf16_attn")
        self.dtype = dtype
        self.ctx = ctx or default_context()
        dev = torch.device("cuda", self.ctx.device)
        k = _dev(keys, torch.float32, dev)
        if k.dim() != 2:
            raise InvalidArgument("keys must be n x d")
        v = _dev(values, torch.float32, dev) if values is not None else None
        if v is not None and v.shape != k.shape:
            raise InvalidArgument("keys and values must have equal n")
        self.n, self.d = int(k.shape[0]), int(k.shape[1])
        h = C.c_void_p()
        if dtype == "f32":
            _check(lib.ra_kv_create(self.ctx.h, _ptr(k), _ptr(v), self.n, self.d, 1, C.byref(h)))
        else:
            _check(lib.ra_kv_create_bf16(self.ctx.h, _ptr(k), _ptr(v), self.n, self.d, 1,
                                         int(dtype == "bf16_attn"), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib.ra_kv_release(self.h)
                self.h = None
        except Exception:
            pass

    def keys_tensor(self) -> torch.Tensor:
        """Zero-copy torch view of the device keys (n x d f32)."""
        return _view_f32(lib.ra_kv_keys_device(self.h), self.n * self.d, self.ctx.device).view(
            self.n, self.d)

    def values_tensor(self) -> torch.Tensor:
        return _view_f32(lib.ra_kv_values_device(self.h), self.n * self.d, self.ctx.device).view(
            self.n, self.d)


def _view_f32(ptr: int, numel: int, device: int) -> torch.Tensor:
    # borrow device memory owned by the library (valid while the owner lives)
    class _Holder:
        __cuda_array_interface__ = {
            "shape": (numel,), "typestr": "<f4", "data": (ptr, False), "version": 2,
            "strides": None}
    return torch.as_tensor(_Holder(), device=f"cuda:{device}")


# ---------------------------------------------------------------------------
# index API  (index.hpp / index_oodgraph.hpp)
# ---------------------------------------------------------------------------
@dataclass
class SearchResult:
    """index.hpp:28-33"""

    ids: np.ndarray
    scores: np.ndarray
    scanned: int = 0
    truncated: bool = False


@dataclass
class OODGraphBuildParams:
    """index_oodgraph.hpp:17-27 (defaults identical)."""

    k_train: int = 32
    max_degree: int = 32
    ef_construction: int = 128
    edge_window: int = 8
    entry_strategy: str = "medoid"   # "medoid" | "maxnorm"
    prune_rule: str = "euclidean"    # "euclidean" | "inner_product"
    default_ef: int = 128

    def to_c(self) -> _capi.BuildParamsC:
        return _capi.BuildParamsC(self.k_train, self.max_degree, self.ef_construction,
                                  self.edge_window, int(self.entry_strategy == "maxnorm"),
                                  int(self.prune_rule == "inner_product"), self.default_ef)


@dataclass
class BuildStats:
    knn_rows: int = 0
    knn_rows_widened: int = 0
    candidate_edges: int = 0
    repair_rounds: int = 0
    repaired_nodes: int = 0
    ms: dict = field(default_factory=dict)


class OODGraph:
    """Attention-aware navigable graph on the device (index_oodgraph.hpp:35-76)."""

    def __init__(self, keys: KVGroup, handle: C.c_void_p, stats: Optional[BuildStats] = None):
        self.keys = keys
        self.h = handle
        self.build_stats = stats

    # -- construction -----------------------------------------------------
    @classmethod
    def from_blob(cls, keys: KVGroup, blob: bytes) -> "OODGraph":
        """OODGraph(keys, blob) (index_oodgraph.hpp:40)."""
        h = C.c_void_p()
        _check(lib.ra_graph_deserialize(keys.ctx.h, keys.h, blob, len(blob), C.byref(h)))
        return cls(keys, h)

    @classmethod
    def load(cls, keys: KVGroup, path) -> "OODGraph":
        try:
            with open(path, "rb") as f:
                blob = f.read()
        except OSError:
            raise GraphError(f"cannot open {path}")
        return cls.from_blob(keys, blob)

    def __del__(self):
        try:
            if self.h:
                lib.ra_graph_free(self.h)
                self.h = None
        except Exception:
            pass

    # -- SearchIndex ------------------------------------------------------------
    def kind(self) -> str:
        return "oodgraph"

    def size(self) -> int:
        return int(lib.ra_graph_size(self.h))

    def memory_bytes(self) -> int:
        return int(lib.ra_graph_memory_bytes(self.h))

    def device_bytes(self) -> int:
        return int(lib.ra_graph_device_bytes(self.h))

    def entry_point(self) -> int:
        return int(lib.ra_graph_entry_point(self.h))

    def max_degree_bound(self) -> int:
        return int(lib.ra_graph_max_degree_bound(self.h))

    def default_ef(self) -> int:
        return int(lib.ra_graph_default_ef(self.h))

    def degree(self, u: int) -> int:
        return int(lib.ra_graph_degree(self.h, u))

    def neighbors(self, u: int) -> np.ndarray:
        cap = self.max_degree_bound()
        out = np.zeros(cap, np.uint32)
        deg = lib.ra_graph_neighbors(self.h, u, out.ctypes.data_as(_capi.c_u32p), cap)
        return out[:deg].copy()

    def reachable_count(self) -> int:
        return int(lib.ra_graph_reachable_count(self.h))

    def serialize(self) -> bytes:
        size = C.c_uint64()
        _check(lib.ra_graph_serialize(self.h, None, 0, C.byref(size)))
        buf = C.create_string_buffer(size.value)
        _check(lib.ra_graph_serialize(self.h, buf, size.value, C.byref(size)))
        return buf.raw[: size.value]

    def save(self, path) -> None:
        with open(path, "wb") as f:
            f.write(self.serialize())

    def search(self, q, k: int, mask=None, ef: Optional[int] = None) -> SearchResult:
        """SearchIndex::search (index.hpp:41-42) for one host query."""
        res = search_batch([self], np.asarray(q, np.float32).reshape(1, -1), k, mask, ef)
        return res[0]


def ood_build(keys: KVGroup, train_queries, params: OODGraphBuildParams = OODGraphBuildParams()
              ) -> OODGraph:
    """ood_build (index_oodgraph.hpp:78-81) on the GPU."""
    dev = torch.device("cuda", keys.ctx.device)
    tq = _dev(train_queries, torch.float32, dev)
    if tq.dim() == 1:
        tq = tq.view(1, -1)
    nq = int(tq.shape[0])
    qdim = int(tq.shape[1]) if tq.dim() == 2 else keys.d
    h = C.c_void_p()
    st = _capi.BuildStatsC()
    bp = params.to_c()
    _check(lib.ra_graph_build(keys.ctx.h, keys.h, _ptr(tq) if nq else None, nq, qdim, 1,
                              C.byref(bp), C.byref(st), C.byref(h)))
    stats = BuildStats(st.knn_rows, st.knn_rows_widened, st.candidate_edges, st.repair_rounds,
                       st.repaired_nodes,
                       dict(knn=st.ms_knn, edges=st.ms_edges, prune=st.ms_prune,
                            entry=st.ms_entry, repair=st.ms_repair, knn_tensor=st.ms_knn_tensor))
    g = OODGraph(keys, h, stats)
    g.default_ef_param = params.default_ef
    return g


@dataclass
class BatchResult:
    """Device-side results of search_batch (torch tensors on the GPU)."""

    ids: torch.Tensor        # [B, k] uint32 viewed as int32 (UINT32_MAX padded)
    scores: torch.Tensor     # [B, k] f32 (NaN padded)
    n_out: torch.Tensor      # [B] int32
    scanned: torch.Tensor    # [B] int64
    truncated: torch.Tensor  # [B] uint8
    expanded: torch.Tensor   # [B] int32

    def __getitem__(self, b) -> SearchResult:
        n = int(self.n_out[b])
        return SearchResult(self.ids[b, :n].cpu().numpy().view(np.uint32).copy(),
                            self.scores[b, :n].cpu().numpy().copy(),
                            int(self.scanned[b]), bool(self.truncated[b]))

    def host(self) -> list:
        ids = self.ids.cpu().numpy().view(np.uint32)
        sc = self.scores.cpu().numpy()
        n = self.n_out.cpu().numpy()
        scn = self.scanned.cpu().numpy()
        tr = self.truncated.cpu().numpy()
        return [SearchResult(ids[b, : n[b]].copy(), sc[b, : n[b]].copy(), int(scn[b]),
                             bool(tr[b])) for b in range(len(n))]


def search_batch(graphs: Sequence[OODGraph], queries, k: int, mask=None,
                 ef: Optional[int] = None, ctx: Optional[Context] = None) -> BatchResult:
    """Batched OODGraph::search: query b walks graphs[b] (or graphs[0] for all)."""
    ctx = ctx or graphs[0].keys.ctx.bind_stream()
    dev = torch.device("cuda", ctx.device)
    q = _dev(queries, torch.float32, dev)
    if q.dim() == 1:
        q = q.view(1, -1)
    B, d = int(q.shape[0]), int(q.shape[1])
    if len(graphs) == 1 and B > 1:
        graphs = list(graphs) * B
    if len(graphs) != B:
        raise InvalidArgument("one graph per query required")
    m = None
    if mask is not None and len(mask) > 0:
        m = _dev(np.asarray(mask, np.uint32).view(np.int32) if not isinstance(mask, torch.Tensor)
                 else mask, torch.int32, dev)
    kk = max(int(k), 1)
    out = BatchResult(
        torch.empty((B, kk), dtype=torch.int32, device=dev),
        torch.empty((B, kk), dtype=torch.float32, device=dev),
        torch.empty(B, dtype=torch.int32, device=dev),
        torch.empty(B, dtype=torch.int64, device=dev),
        torch.empty(B, dtype=torch.uint8, device=dev),
        torch.empty(B, dtype=torch.int32, device=dev))
    arr = (C.c_void_p * B)(*[g.h.value for g in graphs])
    _check(lib.ra_graph_search_batch(
        ctx.h, arr, B, _ptr(q), d, int(k), -1 if ef is None else int(ef), _ptr(m),
        0 if m is None else int(m.numel()), _ptr(out.ids), _ptr(out.scores), _ptr(out.n_out),
        _ptr(out.scanned), _ptr(out.truncated), _ptr(out.expanded)))
    return out


def engine_init(workloads, config: "EngineConfig" = None,
                graph: "OODGraphBuildParams" = None) -> "Engine":
    """engine_init (engine.cpp:23-65) for IndexKind::OODGraph: one KVGroup per
    kv_group_id (uploaded once, shared by its heads), each head's graph built
    on the GPU over its group's keys from its own prefill queries. `workloads`
    are reference-style head bundles (kvd1.HeadWorkload or anything with
    head_id, kv_group_id, prefill_queries, keys, values; vectors as .data or
    arrays). Heads must be ordered by head id with groups contiguous."""
    config = config or EngineConfig()
    graph = graph or OODGraphBuildParams()
    if not workloads:
        raise InvalidArgument("no heads")
    if config.top_k < 1:
        raise InvalidArgument("top_k must be >= 1")
    arr = lambda v: np.asarray(getattr(v, "data", v), np.float32)
    t = arr(workloads[0].keys).shape[0]
    if t == 0:
        raise InvalidArgument("empty context")
    for w in workloads:
        if arr(w.keys).shape[0] != t or arr(w.values).shape[0] != t:
            raise InvalidArgument("context length mismatch across heads")
    groups, gid = [], {}
    for w in workloads:
        if w.kv_group_id not in gid:
            gid[w.kv_group_id] = len(groups)
            groups.append(KVGroup(arr(w.keys), arr(w.values)))
    graphs = [ood_build(groups[gid[w.kv_group_id]], arr(w.prefill_queries), graph)
              for w in workloads]
    return Engine(groups, graphs, config)


class FlatIndex:
    """Exact maximum-inner-product scan on the device (index_flat.hpp:9-22):
    in-order f64 scores of every key, (score desc, id asc) top k, masked ids
    skipped, scanned = n - |mask|. The recall ground truth."""

    def __init__(self, keys: KVGroup):
        if keys.n == 0:
            raise InvalidArgument("empty keys")
        self.keys = keys

    def kind(self) -> str:
        return "flat"

    def size(self) -> int:
        return self.keys.n

    def memory_bytes(self) -> int:
        return 0

    def search_batch(self, queries, k: int, mask=None) -> list:
        ctx = self.keys.ctx.bind_stream()
        dev = torch.device("cuda", ctx.device)
        q = _dev(queries, torch.float32, dev)
        if q.dim() == 1:
            q = q.view(1, -1)
        if int(q.shape[1]) != self.keys.d:
            raise InvalidArgument("query dimension mismatch")
        B = int(q.shape[0])
        m = None
        if mask is not None and len(mask) > 0:
            m = _dev(np.asarray(mask, np.uint32).view(np.int32) if not isinstance(mask, torch.Tensor)
                     else mask, torch.int32, dev)
        kk = max(int(k), 1)
        ids = torch.empty((B, kk), dtype=torch.int32, device=dev)
        sc = torch.empty((B, kk), dtype=torch.float32, device=dev)
        scanned = torch.empty(B, dtype=torch.int64, device=dev)
        _check(lib.ra_flat_search_batch(ctx.h, self.keys.h, B, _ptr(q), int(k), _ptr(m),
                                        0 if m is None else int(m.numel()), _ptr(ids), _ptr(sc),
                                        _ptr(scanned)))
        ih, sh, nh = ids.cpu().numpy().view(np.uint32), sc.cpu().numpy(), scanned.cpu().numpy()
        return [SearchResult(ih[b].copy(), sh[b].copy(), int(nh[b]), False) for b in range(B)]

    def search(self, q, k: int, mask=None, param=None) -> SearchResult:
        """SearchIndex::search (index.hpp:41-42); the flat scan has no knob."""
        return self.search_batch(np.asarray(q, np.float32).reshape(1, -1), k, mask)[0]


@dataclass
class IVFBuildParams:
    """index_ivf.hpp:7-12 (defaults identical)."""

    nlist: int = 0          # 0 = ceil(sqrt(n))
    seed: int = 0
    iters: int = 20
    default_nprobe: int = 8


class IVFIndex:
    """k-means IVF baseline on the device (index_ivf.hpp:17-37)."""

    def __init__(self, keys: KVGroup, params: IVFBuildParams = IVFBuildParams()):
        self.keys = keys
        h = C.c_void_p()
        _check(lib.ra_ivf_build(keys.ctx.h, keys.h, params.nlist, params.seed, params.iters,
                                params.default_nprobe, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib.ra_ivf_free(self.h)
                self.h = None
        except Exception:
            pass

    def kind(self) -> str:
        return "ivf"

    def size(self) -> int:
        return self.keys.n

    def nlist(self) -> int:
        return int(lib.ra_ivf_nlist(self.h))

    def memory_bytes(self) -> int:
        return int(lib.ra_ivf_memory_bytes(self.h))

    def export(self):
        """(centroids [nlist, d] f32, offsets [nlist+1], ids [n]) host copies."""
        nl, d = self.nlist(), self.keys.d
        cent = np.empty((nl, d), np.float32)
        off = np.empty(nl + 1, np.uint32)
        ids = np.empty(self.keys.n, np.uint32)
        _check(lib.ra_ivf_export(self.h, cent.ctypes.data, off.ctypes.data, ids.ctypes.data))
        return cent, off, ids

    def list(self, c: int) -> np.ndarray:
        _, off, ids = self.export()
        return ids[off[c]:off[c + 1]].copy()

    def search_batch(self, queries, k: int, mask=None, nprobe: Optional[int] = None) -> list:
        ctx = self.keys.ctx.bind_stream()
        dev = torch.device("cuda", ctx.device)
        q = _dev(queries, torch.float32, dev)
        if q.dim() == 1:
            q = q.view(1, -1)
        B = int(q.shape[0])
        m = None
        if mask is not None and len(mask) > 0:
            m = _dev(np.asarray(mask, np.uint32).view(np.int32), torch.int32, dev)
        kk = max(int(k), 1)
        ids = torch.empty((B, kk), dtype=torch.int32, device=dev)
        sc = torch.empty((B, kk), dtype=torch.float32, device=dev)
        n_out = torch.empty(B, dtype=torch.int32, device=dev)
        scanned = torch.empty(B, dtype=torch.int64, device=dev)
        tr = torch.empty(B, dtype=torch.uint8, device=dev)
        _check(lib.ra_ivf_search_batch(ctx.h, self.h, B, _ptr(q), int(q.shape[1]), int(k),
                                       -1 if nprobe is None else int(nprobe), _ptr(m),
                                       0 if m is None else int(m.numel()), _ptr(ids), _ptr(sc),
                                       _ptr(n_out), _ptr(scanned), _ptr(tr)))
        ih, sh = ids.cpu().numpy().view(np.uint32), sc.cpu().numpy()
        nh, snh, th = n_out.cpu().numpy(), scanned.cpu().numpy(), tr.cpu().numpy()
        return [SearchResult(ih[b, : nh[b]].copy(), sh[b, : nh[b]].copy(), int(snh[b]), bool(th[b]))
                for b in range(B)]

    def search(self, q, k: int, mask=None, nprobe: Optional[int] = None) -> SearchResult:
        return self.search_batch(np.asarray(q, np.float32).reshape(1, -1), k, mask, nprobe)[0]


def ivf_build(keys: KVGroup, params: IVFBuildParams = IVFBuildParams()) -> IVFIndex:
    """ivf_build (index_ivf.hpp:39-40)."""
    return IVFIndex(keys, params)


def flat_build(keys: KVGroup) -> FlatIndex:
    """flat_build (index_flat.hpp:24)."""
    return FlatIndex(keys)


# ---------------------------------------------------------------------------
# attention  (attention.hpp)
# ---------------------------------------------------------------------------
@dataclass
class PartialAttention:
    """attention.hpp:15-20"""

    out: np.ndarray
    zmax: float = 0.0
    expsum: float = 0.0
    empty: bool = True


@dataclass
class KVPartition:
    static_set: np.ndarray
    dynamic_pool: np.ndarray


def static_partition(t: int, s_init: int, s_local: int) -> KVPartition:
    """attention.cpp:87-100"""
    ns, npool = C.c_uint64(), C.c_uint64()
    _check(lib.ra_static_partition(t, s_init, s_local, None, C.byref(ns), None, C.byref(npool)))
    w = np.zeros(max(ns.value, 1), np.uint32)
    p = np.zeros(max(npool.value, 1), np.uint32)
    _check(lib.ra_static_partition(t, s_init, s_local, w.ctypes.data_as(_capi.c_u32p),
                                   C.byref(ns), p.ctypes.data_as(_capi.c_u32p), C.byref(npool)))
    return KVPartition(w[: ns.value].copy(), p[: npool.value].copy())


def empty_partial(d: int) -> PartialAttention:
    return PartialAttention(np.zeros(d, np.float64))


def partial_attention(q, kv: KVGroup, indices) -> PartialAttention:
    """attention.cpp:102-128 on the GPU."""
    q = np.asarray(q, np.float32).reshape(-1)
    if q.size != kv.d:
        raise InvalidArgument("query dimension mismatch")
    idx = np.asarray(indices, np.uint32).reshape(-1)
    if idx.size == 0:
        raise InvalidArgument("empty index set")
    ctx = kv.ctx.bind_stream()
    dev = torch.device("cuda", ctx.device)
    qd = _dev(q.reshape(1, -1), torch.float32, dev)
    ix = _dev(idx.view(np.int32), torch.int32, dev)
    m = torch.tensor([idx.size], dtype=torch.int32, device=dev)
    out = torch.empty((1, kv.d), dtype=torch.float64, device=dev)
    zm = torch.empty(1, dtype=torch.float64, device=dev)
    es = torch.empty(1, dtype=torch.float64, device=dev)
    _check(lib.ra_partial_attention(ctx.h, kv.h, 1, _ptr(qd), _ptr(ix), int(idx.size), _ptr(m),
                                    _ptr(out), _ptr(zm), _ptr(es)))
    return PartialAttention(out[0].cpu().numpy(), float(zm[0]), float(es[0]), False)


def _merge_dev(pw: PartialAttention, po: PartialAttention):
    d = len(pw.out)
    ctx = default_context()
    dev = torch.device("cuda", ctx.device)
    t = lambda x: torch.tensor(np.asarray(x, np.float64).reshape(1, -1), device=dev)
    ow, oo = t(pw.out), t(po.out)
    zw, sw, zo, so = t([pw.zmax]), t([pw.expsum]), t([po.zmax]), t([po.expsum])
    we = torch.tensor([int(pw.empty)], dtype=torch.uint8, device=dev)
    oe = torch.tensor([int(po.empty)], dtype=torch.uint8, device=dev)
    out = torch.empty((1, d), dtype=torch.float64, device=dev)
    gw = torch.empty(1, dtype=torch.float64, device=dev)
    go = torch.empty(1, dtype=torch.float64, device=dev)
    _check(lib.ra_merge(ctx.h, 1, d, _ptr(ow), _ptr(zw), _ptr(sw), _ptr(we), _ptr(oo), _ptr(zo),
                        _ptr(so), _ptr(oe), _ptr(out), _ptr(gw), _ptr(go)))
    return out[0].cpu().numpy(), float(gw[0]), float(go[0])


def merge_gammas(pw: PartialAttention, po: PartialAttention):
    """attention.cpp:136-147"""
    _, gw, go = _merge_dev(pw, po)
    return gw, go


def merge(pw: PartialAttention, po: PartialAttention) -> np.ndarray:
    """attention.cpp:149-157"""
    return _merge_dev(pw, po)[0]


# ---------------------------------------------------------------------------
# decode engine  (engine.hpp)
# ---------------------------------------------------------------------------
@dataclass
class EngineConfig:
    """engine.hpp:24-39 (decode-path fields)."""

    s_init: int = 128
    s_local: int = 512
    top_k: int = 100
    search_param: Optional[int] = None   # ef override; None = index default


class Engine:
    """engine_init's frozen per-head state + decode_step on the GPU
    (engine.cpp:23-115). groups[g] are the KV groups; graphs[h] is head h's
    graph, built over groups[h // (H // G)]."""

    def __init__(self, groups: Sequence[KVGroup], graphs: Sequence[OODGraph],
                 config: EngineConfig = EngineConfig(), ctx: Optional[Context] = None):
        self.ctx = ctx or groups[0].ctx.bind_stream()
        self.groups, self.graphs, self.config = list(groups), list(graphs), config
        self.H, self.d = len(graphs), groups[0].d
        self.t = groups[0].n
        cfg = _capi.EngineConfigC(config.s_init, config.s_local, config.top_k,
                                  -1 if config.search_param is None else config.search_param)
        g_arr = (C.c_void_p * len(groups))(*[g.h.value for g in groups])
        h_arr = (C.c_void_p * len(graphs))(*[g.h.value for g in graphs])
        h = C.c_void_p()
        _check(lib.ra_engine_create(self.ctx.h, g_arr, len(groups), h_arr, len(graphs),
                                    C.byref(cfg), C.byref(h)))
        self.h = h
        part = static_partition(self.t, config.s_init, config.s_local)
        self.k = min(config.top_k, len(part.dynamic_pool))
        self.w_size = len(part.static_set)
        dev = torch.device("cuda", self.ctx.device)
        self.out = torch.empty((self.H, self.d), dtype=torch.float64, device=dev)
        self.omega = torch.empty((self.H, max(self.k, 1)), dtype=torch.int32, device=dev)
        self.scanned = torch.empty(self.H, dtype=torch.int64, device=dev)

    def __del__(self):
        try:
            if self.h:
                lib.ra_engine_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def decode_step_device(self, q: torch.Tensor):
        """q: [H, d] f32 CUDA tensor -> (out, omega, scanned) device tensors."""
        if (q.dtype != torch.float32 or not q.is_cuda or not q.is_contiguous()
                or tuple(q.shape) != (self.H, self.d)):
            raise InvalidArgument("q must be a contiguous [H, d] float32 CUDA tensor")
        self.ctx.bind_stream()
        _check(lib.ra_engine_step_device(self.h, _ptr(q), _ptr(self.out), _ptr(self.omega),
                                         _ptr(self.scanned)))
        return self.out, self.omega, self.scanned

    def decode_step(self, queries) -> tuple:
        """decode_step (engine.cpp:105-115) from host queries [H, d]:
        returns (out [H,d] f64, omega [H,k] u32, scanned [H] u64) on the host."""
        q = np.ascontiguousarray(queries, np.float32)
        if q.ndim != 2 or q.shape[0] != self.H:
            raise InvalidArgument("one query per head required")
        if q.shape[1] != self.d:  # the C call reads exactly H * d floats
            raise InvalidArgument("query dimension mismatch")
        out = np.empty((self.H, self.d), np.float64)
        om = np.empty((self.H, max(self.k, 1)), np.uint32)
        sc = np.empty(self.H, np.uint64)
        self.ctx.bind_stream()
        _check(lib.ra_engine_step_host(self.h, q.ctypes.data, out.ctypes.data, om.ctypes.data,
                                       sc.ctypes.data))
        return out, om[:, : self.k], sc

    def kernels_per_step(self) -> int:
        """1 for the fused step (search + attention in one kernel), else 3."""
        return int(lib.ra_engine_kernels_per_step(self.h))

    def last_timing(self):
        """(search_ms, attention_ms) of the last step, CUDA events on the ctx stream."""
        a, b = C.c_float(), C.c_float()
        _check(lib.ra_engine_last_timing(self.h, C.byref(a), C.byref(b)))
        return float(a.value), float(b.value)

    def debug_counters(self):
        """{rounds, cycles_pre_expand, cycles_commit, commits} of the last step."""
        out = (C.c_uint64 * 12)()
        _check(lib.ra_engine_debug_counters(self.h, out))
        return dict(zip(("rounds", "cycles_pre_expand", "cycles_commit", "commits", "cy_argmax",
                         "cy_stop", "cy_packet", "cy_add", "cy_select"), list(out)))

    def debug_counters_per_head(self):
        """The same counters per head: uint64 array [H, 12]."""
        out = np.zeros((self.H, 12), dtype=np.uint64)
        _check(lib.ra_engine_debug_counters_per_head(
            self.h, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def last_stats(self):
        s, e = C.c_uint64(), C.c_uint64()
        _check(lib.ra_engine_last_stats(self.h, C.byref(s), C.byref(e)))
        return int(s.value), int(e.value)
