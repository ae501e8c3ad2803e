#!/usr/bin/env python3
"""Profiling driver for the throughput-mode search: one launch of R x 32
queries over config-2 graphs (run under ncu with -k regex:k_graph_search)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RA_SEARCH_KERNEL", "tp")


def main():
    import torch
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    spec = WorkloadSpec(n_ctx=131072, d_model=256, d_head=128, n_heads=32, n_kv_groups=8,
                        seed=7, n_decode=R)
    graphs, dq = [], []
    bp = ra.OODGraphBuildParams(128, 24, 256, 8)
    for g in range(8):
        w = generate_group(spec, g, "cuda")
        kv = ra.KVGroup(w["keys"], w["values"])
        for m in range(4):
            graphs.append(ra.ood_build(kv, w["prefill_q"][m], bp))
            dq.append(w["decode_q"][m])
    Q = torch.stack([dq[h][i] for i in range(R) for h in range(32)]).contiguous()
    gl = [graphs[h] for i in range(R) for h in range(32)]
    W = ra.static_partition(131072, 128, 512).static_set
    for _ in range(3):
        ra.search_batch(gl, Q, 100, W, 128)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
