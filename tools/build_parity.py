#!/usr/bin/env python3
"""Graph-build parity at configs[0] scale: the reference's own ood_build
(oracle/_ref, unmodified sources, all host threads) vs our GPU build on the
same workload (reference generator, seed 7, head 0). Compares the OODG blobs
byte for byte and, if they differ, counts nodes whose adjacency differs and
the entry point. Prints one JSON line (GPU box; minutes of CPU time)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_blob(b):
    import struct
    n, = struct.unpack_from("<Q", b, 8)
    M, = struct.unpack_from("<I", b, 16)
    entry, = struct.unpack_from("<Q", b, 20)
    off, adj = 28, []
    for _ in range(n):
        deg, = struct.unpack_from("<I", b, off)
        off += 4
        adj.append(np.frombuffer(b, "<u8", count=deg, offset=off))
        off += 8 * deg
    return n, M, entry, adj


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    kt, M, efc = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (128, 24, 256)))
    import paper_2409_10516_b200 as ra
    from oracle.ffi import BuildParams, Oracle
    o = Oracle("ref")
    w = o.generate_workload(n, 256, 128, 1, 1, seed=7, n_decode=1, n_threads=os.cpu_count())
    keys, pq = w["keys"][0], w["prefill_q"][0]
    t0 = time.time()
    ref = o.graph_build(keys, pq, BuildParams(k_train=kt, max_degree=M, ef_construction=efc,
                                              edge_window=8), n_threads=os.cpu_count())
    t_ref = time.time() - t0
    kv = ra.KVGroup(keys)
    ra.ood_build(kv, pq, ra.OODGraphBuildParams(kt, M, efc, 8))  # warm-up
    t0 = time.time()
    g = ra.ood_build(kv, pq, ra.OODGraphBuildParams(kt, M, efc, 8))
    t_gpu = time.time() - t0
    ours = g.serialize()
    res = {"n": n, "k_train": kt, "max_degree": M, "ef_construction": efc,
           "ref_build_s": round(t_ref, 2), "ref_threads": os.cpu_count(),
           "gpu_build_s": round(t_gpu, 3), "blob_identical": ours == ref}
    if ours != ref:
        _, _, e1, a1 = parse_blob(ours)
        _, _, e2, a2 = parse_blob(ref)
        res["entry_identical"] = e1 == e2
        res["nodes_with_different_adjacency"] = int(sum(
            not np.array_equal(x, y) for x, y in zip(a1, a2)))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
