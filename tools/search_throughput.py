#!/usr/bin/env python3
"""Throughput of the K6 search at config-2 graphs with many queries in one
launch: R decode queries per head x 32 heads (128K context, ef 128, masked
by the static set W). Prints one JSON line: batch, device ms (CUDA events,
L2 flushed before each launch), algorithmic bytes and GB/s, and a checksum
of the retrieved ids (to compare kernel variants, RA_SEARCH_KERNEL=tp|lat).
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-ctx", type=int, default=131072)
    ap.add_argument("--groups-used", type=int, default=8)
    ap.add_argument("--reps", type=int, nargs="+", default=[1, 8, 32])
    ap.add_argument("--ef", type=int, default=128)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    R = max(a.reps)
    spec = WorkloadSpec(n_ctx=a.n_ctx, d_model=256, d_head=128, n_heads=32, n_kv_groups=8,
                        seed=7, n_decode=R)
    graphs, dq = [], []
    bp = ra.OODGraphBuildParams(128, 24, 256, 8)
    kvs = []
    for g in range(a.groups_used):
        w = generate_group(spec, g, "cuda")
        kv = ra.KVGroup(w["keys"], w["values"])
        kvs.append(kv)
        for m in range(4):
            graphs.append(ra.ood_build(kv, w["prefill_q"][m], bp))
            dq.append(w["decode_q"][m])  # [R, d]
    H = len(graphs)
    W = ra.static_partition(a.n_ctx, 128, 512).static_set
    flush = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
    for r in a.reps:
        Q = torch.stack([dq[h][i] for i in range(r) for h in range(H)]).contiguous()
        gl = [graphs[h] for i in range(r) for h in range(H)]
        ts = []
        for it in range(a.iters + 1):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            res = ra.search_batch(gl, Q, 100, W, a.ef)
            e1.record()
            e1.synchronize()
            if it:
                ts.append(e0.elapsed_time(e1))
        sc = res.scanned.cpu().numpy().astype(np.float64)
        ex = res.expanded.cpu().numpy().astype(np.float64)
        by = float((sc * 128 * 4 + ex * 24 * 4).sum())
        ms = float(np.mean(ts))
        ids = res.ids.cpu().numpy()
        print(json.dumps({"kernel": os.environ.get("RA_SEARCH_KERNEL", "auto"), "batch": len(gl),
                          "ms": round(ms, 4), "us_per_query": round(ms * 1e3 / len(gl), 3),
                          "bytes": by, "GBps": round(by / (ms * 1e-3) / 1e9, 1),
                          "mean_scanned": float(sc.mean()),
                          "ids_sha": hashlib.sha1(ids.tobytes()).hexdigest()[:12]}), flush=True)


if __name__ == "__main__":
    main()
