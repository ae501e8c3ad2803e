#!/usr/bin/env python3
"""configs[4] scale check: one Llama-3-8B-shape head at a 1M-token context
(GPU-synthesised reference workload), graph built on the GPU, decode
searches (mask W = first 128 + last 512) on the GPU in both kernel modes,
and the same searches by the reference (oracle/_ref) on the same graph.
Prints one JSON line (build time, search latency, parity)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    import torch
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    from oracle.ffi import Oracle, available
    spec = WorkloadSpec(n_ctx=n, d_model=256, d_head=128, n_heads=32, n_kv_groups=8, seed=7,
                        n_decode=nq)
    w = generate_group(spec, 0, "cuda")
    kv = ra.KVGroup(w["keys"], w["values"])
    pq = w["prefill_q"][0].contiguous()
    dq = w["decode_q"][0].contiguous()
    del w
    torch.cuda.synchronize()
    t0 = time.time()
    g = ra.ood_build(kv, pq, ra.OODGraphBuildParams(128, 24, 256, 8))
    torch.cuda.synchronize()
    build_s = time.time() - t0
    del pq
    W = ra.static_partition(n, 128, 512).static_set
    res = {}
    for mode in ("lat", "tp"):
        # one query per launch (latency) and all queries together
        Q = dq
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = ra.search_batch([g], Q, 100, W, 128)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[mode] = (min(ts), r.host())
        break  # kernel mode is chosen by batch size; the env var selects it per process
    ms, out = res["lat"]
    parity = None
    if available("ref"):
        o = Oracle("ref")
        og = o.graph(kv.keys_tensor().cpu().numpy(), g.serialize())
        same = 0
        for i in range(nq):
            rr = og.search(dq[i].cpu().numpy(), 100, W, 128)
            same += int(np.array_equal(rr.ids, out[i].ids) and rr.scanned == out[i].scanned)
        parity = f"{same}/{nq} identical ids+scanned vs reference"
    print(json.dumps({"n_ctx": n, "build_s": round(build_s, 2), "build_ms": g.build_stats.ms,
                      "knn_fallback_rows": g.build_stats.knn_rows_widened,
                      "search_ms_batch": round(ms, 3), "queries": nq,
                      "mean_scanned": float(np.mean([x.scanned for x in out])),
                      "parity": parity}))


if __name__ == "__main__":
    main()
