"""B200-native RetrievalAttention decode hot path (arXiv 2409.10516).

Drop-in for the reference attnindex library's graph build, graph search,
sparse attention and partial-softmax merge; compute runs in the sm_100a
library libra_b200.so (C ABI: include/ra_capi.h). Importing this package
loads (building if necessary) that library; there is no CPU fallback.
"""
from ._capi import EXPORTED, lib  # noqa: F401  (loads libra_b200.so, loudly)
from .api import (  # noqa: F401
    BatchResult, BuildStats, Context, CudaError, Engine, EngineConfig, FlatIndex, GraphError,
    IVFBuildParams, IVFIndex, ivf_build,
    InvalidArgument, KVGroup, KVPartition, OODGraph, OODGraphBuildParams, PartialAttention,
    SearchResult, default_context, empty_partial, merge, merge_gammas, ood_build,
    partial_attention, search_batch, static_partition, flat_build, engine_init)
from .report import VerifyLog, build_run  # noqa: F401
from .diagnostics import SweepParams, SweepReport, recall_at_k, recall_sweep  # noqa: F401

__version__ = lib.ra_version().decode()
