"""KVD1 vector files and the workload manifest (reference io.hpp / io.cpp).

Host-side I/O so workloads dumped by the reference (or by a real model)
load straight into KVGroup / OODGraph; byte-identical to the reference's
writer (tests/test_kvd1.py checks against oracle/_ref's save_workloads).

KVD1, little-endian (io.hpp:10-20): "KVD1" | u32 version = 1 | u8 role
(0 = query, 1 = key, 2 = value) | 3 zero bytes | u64 n | u32 d | 4 zero
bytes | n*d f32 row-major. Errors mirror io.cpp:37-96 (std::runtime_error
"kvd1 format error in <path>: <what>") and VectorSet::validate
(workload.cpp:20-27, std::invalid_argument).
"""
from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .api import GraphError, InvalidArgument

MAGIC = b"KVD1"
HEADER = 28
ROLES = {0: "query", 1: "key", 2: "value"}
ROLE_IDS = {v: k for k, v in ROLES.items()}


@dataclass
class VectorSet:
    """types.hpp:18-35: n x d f32 row-major with a role tag."""

    role: int
    data: np.ndarray  # [n, d] float32

    @property
    def n(self) -> int:
        return int(self.data.shape[0])

    @property
    def d(self) -> int:
        return int(self.data.shape[1])

    def validate(self) -> None:
        """workload.cpp:20-27"""
        if self.data.ndim != 2 or self.data.shape[1] < 1:
            raise InvalidArgument("VectorSet.d must be >= 1")
        if not np.isfinite(self.data).all():
            raise InvalidArgument("VectorSet.data contains non-finite entry")


def _fmt(path, what) -> GraphError:
    return GraphError(f"kvd1 format error in {os.fspath(path)}: {what}")


def save_vectors(vs: VectorSet, path) -> None:
    """save_vectors (io.cpp:43-62)."""
    vs.validate()
    hdr = MAGIC + struct.pack("<IB3xQI4x", 1, vs.role, vs.n, vs.d)
    assert len(hdr) == HEADER
    try:
        with open(path, "wb") as f:
            f.write(hdr)
            f.write(np.ascontiguousarray(vs.data, "<f4").tobytes())
    except OSError:
        raise GraphError("cannot open for writing: " + os.fspath(path))


def load_vectors(path) -> VectorSet:
    """load_vectors (io.cpp:64-96)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError:
        raise GraphError("cannot open: " + os.fspath(path))
    if len(raw) < HEADER:
        raise _fmt(path, "truncated header")
    if raw[:4] != MAGIC:
        raise _fmt(path, "bad magic")
    version, = struct.unpack_from("<I", raw, 4)
    if version != 1:
        raise _fmt(path, f"unsupported version {version}")
    role = raw[8]
    if role > 2:
        raise _fmt(path, f"bad role {role}")
    n, = struct.unpack_from("<Q", raw, 12)
    d, = struct.unpack_from("<I", raw, 20)
    if d == 0:
        raise _fmt(path, "d must be >= 1")
    if n > (2 ** 64 - 1) // 4 // d:
        raise _fmt(path, "n*d overflows payload size")
    need = n * d * 4
    if len(raw) - HEADER < need:
        raise _fmt(path, "truncated payload")
    if len(raw) - HEADER > need:
        raise _fmt(path, "trailing bytes after payload")
    data = np.frombuffer(raw, "<f4", count=n * d, offset=HEADER).reshape(n, d).astype(np.float32)
    vs = VectorSet(role, data)
    vs.validate()
    return vs


@dataclass
class ManifestFile:
    head: int
    group: int
    role: str   # "query" | "key" | "value"
    kind: str   # "prefill" | "decode" | "kv"
    path: str


@dataclass
class Manifest:
    """io.hpp:25-38"""

    n_heads: int = 0
    n_kv_groups: int = 0
    d_head: int = 0
    rope_note: str = "synthetic vectors, no positional rotation applied"
    files: List[ManifestFile] = field(default_factory=list)


def save_manifest(m: Manifest, path) -> None:
    """save_manifest (io.cpp:116-120): nlohmann json dump(2) (sorted keys) + newline."""
    obj = {"n_heads": m.n_heads, "n_kv_groups": m.n_kv_groups, "d_head": m.d_head,
           "rope_note": m.rope_note,
           "files": [{"head": f.head, "group": f.group, "role": f.role, "kind": f.kind,
                      "path": f.path} for f in m.files]}
    with open(path, "w") as f:
        f.write(json.dumps(obj, indent=2, sort_keys=True, ensure_ascii=False) + "\n")


def load_manifest(path) -> Manifest:
    """load_manifest (io.cpp:122-141)."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise GraphError("cannot open: " + os.fspath(path))
    m = Manifest(int(j["n_heads"]), int(j["n_kv_groups"]), int(j["d_head"]),
                 j.get("rope_note", ""))
    for f in j["files"]:
        m.files.append(ManifestFile(int(f["head"]), int(f["group"]), f["role"], f["kind"],
                                    f["path"]))
    return m


@dataclass
class HeadWorkload:
    """types.hpp:54-61; keys/values are shared per GQA group (same object)."""

    head_id: int
    kv_group_id: int
    prefill_queries: Optional[VectorSet]
    keys: Optional[VectorSet]
    values: Optional[VectorSet]
    decode_queries: Optional[VectorSet]


def save_workloads(heads: List[HeadWorkload], n_kv_groups: int, dir) -> Manifest:
    """save_workloads (io.cpp:143-177)."""
    os.makedirs(dir, exist_ok=True)
    m = Manifest(len(heads), n_kv_groups, heads[0].keys.d if heads else 0)
    written = [False] * n_kv_groups
    for h in heads:
        name = f"head{h.head_id}_query_prefill.kvd"
        save_vectors(h.prefill_queries, os.path.join(dir, name))
        m.files.append(ManifestFile(h.head_id, h.kv_group_id, "query", "prefill", name))
        name = f"head{h.head_id}_query_decode.kvd"
        save_vectors(h.decode_queries, os.path.join(dir, name))
        m.files.append(ManifestFile(h.head_id, h.kv_group_id, "query", "decode", name))
        if not written[h.kv_group_id]:
            written[h.kv_group_id] = True
            name = f"group{h.kv_group_id}_key.kvd"
            save_vectors(h.keys, os.path.join(dir, name))
            m.files.append(ManifestFile(h.head_id, h.kv_group_id, "key", "kv", name))
            name = f"group{h.kv_group_id}_value.kvd"
            save_vectors(h.values, os.path.join(dir, name))
            m.files.append(ManifestFile(h.head_id, h.kv_group_id, "value", "kv", name))
    save_manifest(m, os.path.join(dir, "manifest.json"))
    return m


def load_workloads(manifest_path) -> List[HeadWorkload]:
    """load_workloads (io.cpp:179-220): heads of a group share one key and one
    value set (object identity preserved)."""
    m = load_manifest(manifest_path)
    d = os.path.dirname(os.fspath(manifest_path))
    gk: List[Optional[VectorSet]] = [None] * m.n_kv_groups
    gv: List[Optional[VectorSet]] = [None] * m.n_kv_groups
    heads = [HeadWorkload(h, 0, None, None, None, None) for h in range(m.n_heads)]
    for f in m.files:
        if f.role == "query":
            if f.head >= m.n_heads:
                raise GraphError("manifest head out of range: " + f.path)
            vs = load_vectors(os.path.join(d, f.path))
            heads[f.head].kv_group_id = f.group
            if f.kind == "prefill":
                heads[f.head].prefill_queries = vs
            elif f.kind == "decode":
                heads[f.head].decode_queries = vs
            else:
                raise GraphError("manifest query kind unknown: " + f.kind)
        elif f.role in ("key", "value"):
            if f.group >= m.n_kv_groups:
                raise GraphError("manifest group out of range: " + f.path)
            vs = load_vectors(os.path.join(d, f.path))
            (gk if f.role == "key" else gv)[f.group] = vs
        else:
            raise GraphError("manifest role unknown: " + f.role)
    for h in heads:
        if h.kv_group_id >= m.n_kv_groups:
            raise GraphError("manifest missing key/value file for group " + str(h.kv_group_id))
        h.keys, h.values = gk[h.kv_group_id], gv[h.kv_group_id]
        if h.keys is None or h.values is None:
            raise GraphError("manifest missing key/value file for group " + str(h.kv_group_id))
    return heads
