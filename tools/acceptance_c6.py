#!/usr/bin/env python3
"""Acceptance criterion 6 (reference tests/acceptance/acceptance.cpp:338-410)
on the GPU: graph vs IVF retrieval cost at matched recall@100, n_ctx 65536,
seeds 7/8/9 (reference generator via oracle/_ref so the inputs are the
reference's own), recall against the GPU FlatIndex (diagnostics.cpp:143-194
recall_sweep: unmasked, scan fraction = scanned / n). Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2409_10516_b200 as ra
    from oracle.ffi import Oracle
    o = Oracle("ref")
    n, k = 65536, 100
    graph_grid = [100, 128, 160, 192, 256, 320]
    ivf_grid = [4, 8, 16, 24, 32, 48, 64, 96, 128, 192]
    g_rec, g_scan = np.zeros(len(graph_grid)), np.zeros(len(graph_grid))
    v_rec, v_scan = np.zeros(len(ivf_grid)), np.zeros(len(ivf_grid))
    t0 = time.time()
    for seed in (7, 8, 9):
        w = o.generate_workload(n, 256, 128, 1, 1, seed=seed, n_decode=256,
                                n_threads=os.cpu_count())
        kv = ra.KVGroup(w["keys"][0])
        dq = w["decode_q"][0]
        truth = [set(r.ids.tolist()) for r in ra.FlatIndex(kv).search_batch(dq, k)]
        g = ra.ood_build(kv, w["prefill_q"][0], ra.OODGraphBuildParams(128, 24, 256, 8))
        for i, ef in enumerate(graph_grid):
            res = ra.search_batch([g], dq, k, None, ef).host()
            g_rec[i] += np.mean([len(truth[j] & set(r.ids.tolist())) / k
                                 for j, r in enumerate(res)]) / 3
            g_scan[i] += np.mean([r.scanned / n for r in res]) / 3
        ix = ra.IVFIndex(kv, ra.IVFBuildParams(nlist=256, seed=seed))
        for i, npb in enumerate(ivf_grid):
            res = ix.search_batch(dq, k, None, npb)
            v_rec[i] += np.mean([len(truth[j] & set(r.ids.tolist())) / k
                                 for j, r in enumerate(res)]) / 3
            v_scan[i] += np.mean([r.scanned / n for r in res]) / 3
    gmin = min([s for r, s in zip(g_rec, g_scan) if r >= 0.95], default=float("inf"))
    vmin = min([s for r, s in zip(v_rec, v_scan) if r >= 0.95], default=float("inf"))
    print(json.dumps({
        "graph": [{"ef": e, "recall": round(float(r), 4), "scan": round(float(s), 5)}
                  for e, r, s in zip(graph_grid, g_rec, g_scan)],
        "ivf": [{"nprobe": p, "recall": round(float(r), 4), "scan": round(float(s), 5)}
                for p, r, s in zip(ivf_grid, v_rec, v_scan)],
        "graph_min_scan_at_recall_0.95": gmin, "ivf_min_scan_at_recall_0.95": vmin,
        "ratio": vmin / gmin if np.isfinite(gmin) else None,
        "criterion": {"graph <= 0.05": bool(gmin <= 0.05), "ivf reaches 0.95": bool(np.isfinite(vmin)),
                      "ivf >= 4x graph": bool(vmin >= 4 * gmin)},
        "wall_s": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
