"""ctypes bindings for the CPU checkers. TEST INFRASTRUCTURE ONLY.

Two backends with one numpy-facing API:
  * ``Oracle("port")`` -> oracle/_build/liboracle.so, our C restatement
    (oracle/ra_oracle.c), buildable anywhere with gcc;
  * ``Oracle("ref")``  -> oracle/_ref/libattnindex_ref.so, the unmodified
    reference sources (/root/reference/proj/src) built by oracle/Makefile;
  * ``Oracle("dropin")`` -> oracle/_ref/libattnindex_dropin.so, the same
    reference library with src/index_oodgraph.cpp, attention.cpp and
    engine.cpp replaced by the drop-in TUs (paper_2409_10516_b200/host/) over
    libra_b200.so: the reference's own API, running on the GPU backend.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import
this module. Errors raise ``OracleError`` carrying the reference's message.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libattnindex_ref.so")
DROPIN_LIB = os.path.join(HERE, "_ref", "libattnindex_dropin.so")
REF_SRC = "/root/reference/proj"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    pass


def build(ref: bool = True) -> None:
    """Compile the checker(s). The reference build needs /root/reference."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def available(kind: str) -> bool:
    return os.path.exists({"port": PORT_LIB, "ref": REF_LIB, "dropin": DROPIN_LIB}[kind])


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class Search:
    ids: np.ndarray
    scores: np.ndarray
    scanned: int
    truncated: bool
    expanded: int | None = None


@dataclass
class BuildParams:
    """OODGraphBuildParams (index_oodgraph.hpp:17-27) defaults."""

    k_train: int = 32
    max_degree: int = 32
    ef_construction: int = 128
    edge_window: int = 8
    entry_maxnorm: bool = False
    prune_inner_product: bool = False
    default_ef: int = 128


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind not in ("port", "ref", "dropin"):
            raise ValueError(kind)
        self.backend = kind
        kind = "ref" if kind == "dropin" else kind  # same C entry points
        self.kind = kind
        path = {"port": PORT_LIB, "ref": REF_LIB, "dropin": DROPIN_LIB}[self.backend]
        if not os.path.exists(path):
            build(ref=(kind == "ref"))
        self.lib = C.CDLL(path)
        self.p = "ora_" if kind == "port" else "ref_"
        self._decl()

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _decl(self):
        L = self._f
        L("last_error").restype = C.c_char_p
        L("splitmix64").restype = C.c_uint64
        L("splitmix64").argtypes = [u64p]
        L("generate_workload").argtypes = (
            [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
             C.c_double, C.c_double, C.c_uint64]
            + ([C.c_int] if self.kind == "ref" else []) + [f32p] * 4)
        L("graph_search").argtypes = (
            ([C.c_void_p, f32p, C.c_uint32, C.c_uint64, u32p, C.c_uint64, C.c_int64,
              u32p, f32p, u64p, u64p, u8p])
            if self.kind == "ref" else
            ([C.c_void_p, f32p, f32p, C.c_uint64, u32p, C.c_uint64, C.c_int64,
              u32p, f32p, u64p, u64p, u8p, u64p]))
        L("flat_search").argtypes = [f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint64, u32p,
                                     C.c_uint64, u32p, f32p, u64p, u64p]
        L("partial_attention").argtypes = [f32p, f32p, f32p, C.c_uint64, C.c_uint32, u32p,
                                           C.c_uint64, f64p, f64p, f64p]
        L("merge").argtypes = [C.c_uint32, f64p, C.c_double, C.c_double, C.c_int, f64p,
                               C.c_double, C.c_double, C.c_int, f64p, f64p, f64p]
        L("static_partition").argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u32p, u64p,
                                          u32p, u64p]
        if self.kind == "ref":
            L("graph_build").argtypes = [f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint64,
                                         C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_int, C.c_int, C.c_uint32, C.c_int,
                                         C.POINTER(C.c_void_p)]
            L("graph_from_blob").argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_char_p,
                                             C.c_uint64, C.POINTER(C.c_void_p)]
            L("graph_serialize").argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, u64p]
            L("graph_free").argtypes = [C.c_void_p]
            L("graph_entry").restype = C.c_uint64
            L("graph_entry").argtypes = [C.c_void_p]
            L("engine_create").argtypes = [f32p, f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                           C.c_uint32, C.c_char_p, u64p, C.c_uint64,
                                           C.c_uint64, C.c_uint32, C.c_int64, C.c_int,
                                           C.POINTER(C.c_void_p)]
            L("engine_step").argtypes = [C.c_void_p, f32p, C.c_uint64, f64p, u32p, u64p]
            L("engine_from_workload").argtypes = (
                [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64] + [C.c_uint32] * 4
                + [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int64, C.c_int, C.c_int]
                + [f32p, f32p, f32p, f64p, f64p, C.POINTER(C.c_void_p)])
            L("engine_graph_serialize").argtypes = [C.c_void_p, C.c_uint32, C.c_char_p,
                                                    C.c_uint64, u64p]
            L("engine_free").argtypes = [C.c_void_p]
        else:
            L("training_knn").argtypes = [f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint64,
                                          C.c_uint32, u32p]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self._f("last_error")().decode())

    # ---- util ------------------------------------------------------------
    def splitmix64(self, state: int, count: int) -> list[int]:
        s = C.c_uint64(state)
        return [self._f("splitmix64")(C.byref(s)) for _ in range(count)]

    # ---- workload ----------------------------------------------------------
    def generate_workload(self, n_ctx, d_model=256, d_head=128, n_heads=1, n_kv_groups=1,
                          seed=7, ood_strength=2.0, concentration=12.0, n_decode=256,
                          n_threads=1):
        pq = np.zeros((n_heads, n_ctx, d_head), np.float32)
        dq = np.zeros((n_heads, n_decode, d_head), np.float32)
        K = np.zeros((n_kv_groups, n_ctx, d_head), np.float32)
        V = np.zeros((n_kv_groups, n_ctx, d_head), np.float32)
        args = [n_ctx, d_model, d_head, n_heads, n_kv_groups, seed, ood_strength,
                concentration, n_decode]
        if self.kind == "ref":
            args.append(n_threads)
        self._check(self._f("generate_workload")(*args, _ptr(pq, f32p), _ptr(dq, f32p),
                                                 _ptr(K, f32p), _ptr(V, f32p)))
        return dict(prefill_q=pq, decode_q=dq, keys=K, values=V)

    # ---- graph -------------------------------------------------------------
    def graph_build(self, keys, train_q, params: BuildParams = BuildParams(), n_threads=1):
        """Returns the OODG v1 blob (bytes)."""
        keys = np.ascontiguousarray(keys, np.float32)
        tq = np.ascontiguousarray(train_q, np.float32).reshape(-1, keys.shape[1])
        p = params
        if self.kind == "ref":
            h = C.c_void_p()
            self._check(self._f("graph_build")(
                _ptr(keys, f32p), keys.shape[0], keys.shape[1], _ptr(tq, f32p), tq.shape[0],
                p.k_train, p.max_degree, p.ef_construction, p.edge_window,
                int(p.entry_maxnorm), int(p.prune_inner_product), p.default_ef, n_threads,
                C.byref(h)))
            try:
                return self._ref_serialize(h)
            finally:
                self._f("graph_free")(h)
        g = _OraGraph()
        bp = _OraBuildParams(p.k_train, p.max_degree, p.ef_construction, p.edge_window,
                             int(p.entry_maxnorm), int(p.prune_inner_product), p.default_ef)
        self.lib.ora_graph_build.argtypes = [f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint64,
                                             C.POINTER(_OraBuildParams),
                                             C.POINTER(_OraGraph)]
        self._check(self.lib.ora_graph_build(_ptr(keys, f32p), keys.shape[0], keys.shape[1],
                                             _ptr(tq, f32p), tq.shape[0], C.byref(bp),
                                             C.byref(g)))
        try:
            return _ora_serialize(self.lib, g)
        finally:
            self.lib.ora_graph_free(C.byref(g))

    def _ref_serialize(self, h) -> bytes:
        size = C.c_uint64()
        self._check(self._f("graph_serialize")(h, None, 0, C.byref(size)))
        buf = C.create_string_buffer(size.value)
        self._check(self._f("graph_serialize")(h, buf, size.value, C.byref(size)))
        return buf.raw[: size.value]

    def training_knn(self, keys, train_q, k_train):
        assert self.kind == "port"
        keys = np.ascontiguousarray(keys, np.float32)
        tq = np.ascontiguousarray(train_q, np.float32)
        kt = min(k_train, keys.shape[0])
        out = np.zeros((tq.shape[0], kt), np.uint32)
        self._f("training_knn")(_ptr(keys, f32p), keys.shape[0], keys.shape[1],
                                _ptr(tq, f32p), tq.shape[0], kt, _ptr(out, u32p))
        return out

    def graph(self, keys, blob: bytes, default_ef: int = 128):
        return OracleGraph(self, np.ascontiguousarray(keys, np.float32), blob, default_ef)

    # ---- flat / attention --------------------------------------------------
    def flat_search(self, keys, q, k, mask=None):
        keys = np.ascontiguousarray(keys, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        m = np.ascontiguousarray(mask if mask is not None else [], np.uint32)
        ids = np.zeros(max(k, 1), np.uint32)
        sc = np.zeros(max(k, 1), np.float32)
        n_out, scanned = C.c_uint64(), C.c_uint64()
        self._check(self._f("flat_search")(_ptr(keys, f32p), keys.shape[0], keys.shape[1],
                                           _ptr(q, f32p), k, _ptr(m, u32p), m.size,
                                           _ptr(ids, u32p), _ptr(sc, f32p), C.byref(n_out),
                                           C.byref(scanned)))
        return Search(ids[: n_out.value].copy(), sc[: n_out.value].copy(), scanned.value, False)

    def partial_attention(self, q, keys, values, idx):
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        idx = np.ascontiguousarray(idx, np.uint32)
        out = np.zeros(keys.shape[1], np.float64)
        zmax, expsum = C.c_double(), C.c_double()
        self._check(self._f("partial_attention")(
            _ptr(q, f32p), _ptr(keys, f32p), _ptr(values, f32p), keys.shape[0], keys.shape[1],
            _ptr(idx, u32p), idx.size, _ptr(out, f64p), C.byref(zmax), C.byref(expsum)))
        return out, zmax.value, expsum.value

    def merge(self, pw, po, d):
        """pw/po: (out, zmax, expsum) or None for empty_partial."""
        zero = np.zeros(d, np.float64)
        ow, zw, sw = pw if pw is not None else (zero, 0.0, 0.0)
        oo, zo, so = po if po is not None else (zero, 0.0, 0.0)
        ow = np.ascontiguousarray(ow, np.float64)
        oo = np.ascontiguousarray(oo, np.float64)
        out = np.zeros(d, np.float64)
        gw, go = C.c_double(), C.c_double()
        self._check(self._f("merge")(d, _ptr(ow, f64p), zw, sw, int(pw is None),
                                     _ptr(oo, f64p), zo, so, int(po is None),
                                     _ptr(out, f64p), C.byref(gw), C.byref(go)))
        return out, gw.value, go.value

    def static_partition(self, t, s_init=128, s_local=512):
        ns, npool = C.c_uint64(), C.c_uint64()
        self._check(self._f("static_partition")(t, s_init, s_local, None, C.byref(ns),
                                                None, C.byref(npool)))
        w = np.zeros(max(ns.value, 1), np.uint32)
        pool = np.zeros(max(npool.value, 1), np.uint32)
        self._check(self._f("static_partition")(t, s_init, s_local, _ptr(w, u32p),
                                                C.byref(ns), _ptr(pool, u32p),
                                                C.byref(npool)))
        return w[: ns.value].copy(), pool[: npool.value].copy()

    # ---- reference decode engine (cpu baseline) ----------------------------
    def engine(self, keys, values, blobs, s_init=128, s_local=512, top_k=100, ef=-1,
               n_threads=1):
        assert self.kind == "ref"
        return RefEngine(self, keys, values, blobs, s_init, s_local, top_k, ef, n_threads)


    def engine_from_workload(self, n_ctx, n_heads=32, n_kv_groups=8, seed=7, n_decode=64,
                             params: "BuildParams" = None, s_init=128, s_local=512,
                             top_k=100, ef=-1, n_threads=1, build_workers=1,
                             keep_kv=False):
        """The reference's own setup: generate_workload + engine_init
        (OODGraph). Returns (engine, decode_q [H, n_decode, d], keys, values,
        ms_gen, ms_build); keys/values are None unless keep_kv."""
        assert self.kind == "ref"
        p = params or BuildParams()
        d = 128
        dq = np.zeros((n_heads, n_decode, d), np.float32)
        K = np.zeros((n_kv_groups, n_ctx, d), np.float32) if keep_kv else None
        V = np.zeros((n_kv_groups, n_ctx, d), np.float32) if keep_kv else None
        h = C.c_void_p()
        mg, mb = C.c_double(), C.c_double()
        self._check(self._f("engine_from_workload")(
            n_ctx, n_heads, n_kv_groups, seed, n_decode, p.k_train, p.max_degree,
            p.ef_construction, p.edge_window, s_init, s_local, top_k, ef, n_threads,
            build_workers, _ptr(dq, f32p), _ptr(K, f32p) if keep_kv else None,
            _ptr(V, f32p) if keep_kv else None, C.byref(mg), C.byref(mb), C.byref(h)))
        eng = RefEngine.__new__(RefEngine)
        eng.o, eng.h, eng.H, eng.d, eng.top_k = self, h, n_heads, d, top_k
        eng.keys = eng.values = None
        return eng, dq, K, V, mg.value, mb.value


class _OraGraph(C.Structure):
    _fields_ = [("n", C.c_uint64), ("d", C.c_uint32), ("max_degree", C.c_uint32),
                ("default_ef", C.c_uint32), ("entry", C.c_uint64),
                ("offsets", u64p), ("adjacency", u32p)]


class _OraBuildParams(C.Structure):
    _fields_ = [("k_train", C.c_uint32), ("max_degree", C.c_uint32),
                ("ef_construction", C.c_uint32), ("edge_window", C.c_uint32),
                ("entry_maxnorm", C.c_int), ("prune_inner_product", C.c_int),
                ("default_ef", C.c_uint32)]


def _ora_serialize(lib, g) -> bytes:
    lib.ora_graph_serialize.restype = C.c_uint64
    lib.ora_graph_serialize.argtypes = [C.POINTER(_OraGraph), C.c_char_p, C.c_uint64]
    size = lib.ora_graph_serialize(C.byref(g), None, 0)
    buf = C.create_string_buffer(size)
    lib.ora_graph_serialize(C.byref(g), buf, size)
    return buf.raw[:size]


class OracleGraph:
    """A searchable graph held by either backend (loaded from an OODG blob)."""

    def __init__(self, o: Oracle, keys, blob: bytes, default_ef: int):
        self.o, self.keys = o, keys
        self.n, self.d = keys.shape
        if o.kind == "ref":
            self.h = C.c_void_p()
            o._check(o._f("graph_from_blob")(_ptr(keys, f32p), self.n, self.d, blob,
                                              len(blob), C.byref(self.h)))
        else:
            self.g = _OraGraph()
            o.lib.ora_graph_from_blob.argtypes = [C.c_uint64, C.c_uint32, C.c_char_p,
                                                  C.c_uint64, C.POINTER(_OraGraph)]
            o._check(o.lib.ora_graph_from_blob(self.n, self.d, blob, len(blob),
                                               C.byref(self.g)))
            self.g.default_ef = default_ef

    def close(self):
        if self.o.kind == "ref":
            if self.h:
                self.o._f("graph_free")(self.h)
                self.h = C.c_void_p()
        elif self.g.offsets:
            self.o.lib.ora_graph_free(C.byref(self.g))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, q, k, mask=None, ef=None) -> Search:
        q = np.ascontiguousarray(q, np.float32)
        m = np.ascontiguousarray(mask if mask is not None else [], np.uint32)
        ef_arg = -1 if ef is None else int(ef)
        cap = max(k, 1)
        ids = np.zeros(cap, np.uint32)
        sc = np.zeros(cap, np.float32)
        n_out, scanned, tr = C.c_uint64(), C.c_uint64(), C.c_uint8()
        if self.o.kind == "ref":
            self.o._check(self.o._f("graph_search")(
                self.h, _ptr(q, f32p), q.size, k, _ptr(m, u32p), m.size, ef_arg,
                _ptr(ids, u32p), _ptr(sc, f32p), C.byref(n_out), C.byref(scanned),
                C.byref(tr)))
            return Search(ids[: n_out.value].copy(), sc[: n_out.value].copy(),
                          scanned.value, bool(tr.value))
        if q.size != self.d:
            raise OracleError("query dimension mismatch")
        exp = C.c_uint64()
        self.o._check(self.o.lib.ora_graph_search(
            C.byref(self.g), _ptr(self.keys, f32p), _ptr(q, f32p), k, _ptr(m, u32p), m.size,
            ef_arg, _ptr(ids, u32p), _ptr(sc, f32p), C.byref(n_out), C.byref(scanned),
            C.byref(tr), C.byref(exp)))
        return Search(ids[: n_out.value].copy(), sc[: n_out.value].copy(), scanned.value,
                      bool(tr.value), exp.value)


class RefEngine:
    """engine.cpp decode_step over blob-loaded graphs (ref backend only)."""

    def __init__(self, o, keys, values, blobs, s_init, s_local, top_k, ef, n_threads):
        self.o = o
        self.keys = np.ascontiguousarray(keys, np.float32)    # [G, t, d]
        self.values = np.ascontiguousarray(values, np.float32)
        G, t, d = self.keys.shape
        H = len(blobs)
        self.H, self.d, self.top_k = H, d, top_k
        sizes = np.array([len(b) for b in blobs], np.uint64)
        allb = b"".join(blobs)
        self.h = C.c_void_p()
        o._check(o._f("engine_create")(_ptr(self.keys, f32p), _ptr(self.values, f32p), t, d,
                                       H, G, allb, _ptr(sizes, u64p), s_init, s_local, top_k,
                                       ef, n_threads, C.byref(self.h)))

    def step(self, q, step=0):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros((self.H, self.d), np.float64)
        om = np.zeros((self.H, self.top_k), np.uint32)
        sc = np.zeros(self.H, np.uint64)
        self.o._check(self.o._f("engine_step")(self.h, _ptr(q, f32p), step, _ptr(out, f64p),
                                               _ptr(om, u32p), _ptr(sc, u64p)))
        return out, om, sc

    def graph_blob(self, h: int) -> bytes:
        size = C.c_uint64()
        self.o._check(self.o._f("engine_graph_serialize")(self.h, h, None, 0, C.byref(size)))
        buf = C.create_string_buffer(size.value)
        self.o._check(self.o._f("engine_graph_serialize")(self.h, h, buf, size.value,
                                                          C.byref(size)))
        return buf.raw[: size.value]

    def __del__(self):
        try:
            self.o._f("engine_free")(self.h)
        except Exception:
            pass
