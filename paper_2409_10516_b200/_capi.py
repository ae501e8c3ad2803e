"""ctypes declarations for libra_b200.so (include/ra_capi.h).

This is the only place Python touches the C ABI; everything above it
(paper_2409_10516_b200.api) is the host-side mirror of the reference's C++
interface. The library is loaded eagerly and a missing or stale build is an
ImportError — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

c_u8p = C.POINTER(C.c_uint8)
c_u32p = C.POINTER(C.c_uint32)
c_u64p = C.POINTER(C.c_uint64)
c_f32p = C.POINTER(C.c_float)
c_f64p = C.POINTER(C.c_double)
c_vp = C.c_void_p

RA_OK, RA_ERR_INVALID_ARGUMENT, RA_ERR_RUNTIME, RA_ERR_CUDA, RA_ERR_CAPACITY = range(5)


class BuildParamsC(C.Structure):
    _fields_ = [("k_train", C.c_uint32), ("max_degree", C.c_uint32),
                ("ef_construction", C.c_uint32), ("edge_window", C.c_uint32),
                ("entry_maxnorm", C.c_int32), ("prune_inner_product", C.c_int32),
                ("default_ef", C.c_uint32)]


class BuildStatsC(C.Structure):
    _fields_ = [("knn_rows", C.c_uint64), ("knn_rows_widened", C.c_uint64),
                ("candidate_edges", C.c_uint64), ("repair_rounds", C.c_uint64),
                ("repaired_nodes", C.c_uint64), ("ms_knn", C.c_double),
                ("ms_edges", C.c_double), ("ms_prune", C.c_double), ("ms_entry", C.c_double),
                ("ms_repair", C.c_double), ("ms_knn_tensor", C.c_double)]


class EngineConfigC(C.Structure):
    _fields_ = [("s_init", C.c_uint64), ("s_local", C.c_uint64), ("top_k", C.c_uint32),
                ("ef", C.c_int64)]


_SIGS = {
    "ra_last_error": (C.c_char_p, []),
    "ra_version": (C.c_char_p, []),
    "ra_ctx_create": (C.c_int, [C.c_int, C.POINTER(c_vp)]),
    "ra_ctx_destroy": (None, [c_vp]),
    "ra_ctx_set_stream": (C.c_int, [c_vp, c_vp]),
    "ra_ctx_synchronize": (C.c_int, [c_vp]),
    "ra_ctx_set_search_kernel": (C.c_int, [c_vp, C.c_char_p]),
    "ra_kv_create": (C.c_int, [c_vp, c_vp, c_vp, C.c_uint64, C.c_uint32, C.c_int,
                               C.POINTER(c_vp)]),
    "ra_kv_create_bf16": (C.c_int, [c_vp, c_vp, c_vp, C.c_uint64, C.c_uint32, C.c_int,
                                    C.c_int, C.POINTER(c_vp)]),
    "ra_kv_is_bf16": (C.c_int, [c_vp]),
    "ra_kv_retain": (None, [c_vp]),
    "ra_kv_release": (None, [c_vp]),
    "ra_kv_size": (C.c_uint64, [c_vp]),
    "ra_kv_dim": (C.c_uint32, [c_vp]),
    "ra_kv_keys_device": (c_vp, [c_vp]),
    "ra_kv_values_device": (c_vp, [c_vp]),
    "ra_build_params_default": (None, [C.POINTER(BuildParamsC)]),
    "ra_graph_build": (C.c_int, [c_vp, c_vp, c_vp, C.c_uint64, C.c_uint32, C.c_int,
                                 C.POINTER(BuildParamsC), C.POINTER(BuildStatsC),
                                 C.POINTER(c_vp)]),
    "ra_graph_deserialize": (C.c_int, [c_vp, c_vp, C.c_char_p, C.c_uint64, C.POINTER(c_vp)]),
    "ra_graph_serialize": (C.c_int, [c_vp, C.c_char_p, C.c_uint64, c_u64p]),
    "ra_graph_free": (None, [c_vp]),
    "ra_graph_size": (C.c_uint64, [c_vp]),
    "ra_graph_entry_point": (C.c_uint64, [c_vp]),
    "ra_graph_max_degree_bound": (C.c_uint32, [c_vp]),
    "ra_graph_default_ef": (C.c_uint32, [c_vp]),
    "ra_graph_degree": (C.c_uint32, [c_vp, C.c_uint64]),
    "ra_graph_neighbors": (C.c_uint32, [c_vp, C.c_uint64, c_u32p, C.c_uint32]),
    "ra_graph_reachable_count": (C.c_uint64, [c_vp]),
    "ra_graph_memory_bytes": (C.c_uint64, [c_vp]),
    "ra_graph_device_bytes": (C.c_uint64, [c_vp]),
    "ra_graph_csr": (C.c_int, [c_vp, c_u64p, c_u32p]),
    "ra_graph_search_host": (C.c_int, [c_vp, c_vp, c_f32p, C.c_uint32, C.c_uint32, C.c_int64, c_u32p,
                                       C.c_uint64, c_u32p, c_f32p, c_u32p, c_u64p, c_u8p]),
    "ra_graph_search_batch": (C.c_int, [c_vp, C.POINTER(c_vp), C.c_uint32, c_vp, C.c_uint32,
                                        C.c_uint32, C.c_int64, c_vp, C.c_uint64, c_vp, c_vp,
                                        c_vp, c_vp, c_vp, c_vp]),
    "ra_flat_search_batch": (C.c_int, [c_vp, c_vp, C.c_uint32, c_vp, C.c_uint32, c_vp,
                                       C.c_uint64, c_vp, c_vp, c_vp]),
    "ra_static_partition": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, c_u32p, c_u64p,
                                      c_u32p, c_u64p]),
    "ra_partial_attention": (C.c_int, [c_vp, c_vp, C.c_uint32, c_vp, c_vp, C.c_uint32, c_vp,
                                       c_vp, c_vp, c_vp]),
    "ra_merge": (C.c_int, [c_vp, C.c_uint32, C.c_uint32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                           c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ra_ivf_build": (C.c_int, [c_vp, c_vp, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                               C.POINTER(c_vp)]),
    "ra_ivf_free": (None, [c_vp]),
    "ra_ivf_nlist": (C.c_uint32, [c_vp]),
    "ra_ivf_default_nprobe": (C.c_uint32, [c_vp]),
    "ra_ivf_export": (C.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "ra_ivf_memory_bytes": (C.c_uint64, [c_vp]),
    "ra_ivf_search_batch": (C.c_int, [c_vp, c_vp, C.c_uint32, c_vp, C.c_uint32, C.c_uint32,
                                      C.c_int64, c_vp, C.c_uint64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ra_engine_create": (C.c_int, [c_vp, C.POINTER(c_vp), C.c_uint32, C.POINTER(c_vp),
                                   C.c_uint32, C.POINTER(EngineConfigC), C.POINTER(c_vp)]),
    "ra_engine_destroy": (None, [c_vp]),
    "ra_engine_step_device": (C.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ra_engine_step_host": (C.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ra_engine_last_stats": (C.c_int, [c_vp, c_u64p, c_u64p]),
    "ra_engine_last_timing": (C.c_int, [c_vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "ra_engine_kernels_per_step": (C.c_uint32, [c_vp]),
    "ra_engine_k": (C.c_uint32, [c_vp]),
    "ra_kv_attach_values": (C.c_int, [c_vp, c_vp, c_vp, C.c_uint64, C.c_int]),
    "ra_kv_has_values": (C.c_int, [c_vp]),
    "ra_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(c_vp)]),
    "ra_host_free": (None, [c_vp]),
    "ra_partial_attention_host": (C.c_int, [c_vp, c_vp, C.c_uint32, c_vp, C.c_uint64, c_vp,
                                            C.c_uint64, C.c_uint32, c_vp, C.c_uint64, c_vp,
                                            c_vp, c_vp]),
    "ra_merge_host": (C.c_int, [c_vp, C.c_uint32, c_vp, C.c_double, C.c_double, C.c_int, c_vp,
                                C.c_double, C.c_double, C.c_int, c_vp, c_vp, c_vp]),
    "ra_engine_debug_counters": (C.c_int, [c_vp, c_u64p]),
    "ra_engine_debug_counters_per_head": (C.c_int, [c_vp, c_u64p]),
}

EXPORTED = tuple(_SIGS)


def load(path: str | None = None) -> C.CDLL:
    path = path or _build.LIB
    if not os.path.exists(path) or _build.stale():
        try:
            _build.build()
        except Exception as e:  # loud: the product has no CPU path
            raise ImportError(f"libra_b200.so is missing and could not be built: {e}") from e
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = load()
