#!/usr/bin/env python3
"""Profiling driver: config-2 decode steps on a subset of KV groups.

  ncu --set full --import-source on -k regex:k_graph_search -s 2 -c 1 \
      -o gpurun_out/search python tools/profile_step.py --groups-used 2

Builds `--groups-used` KV groups (4 heads each) at 128K on the GPU and runs
`--steps` decode steps through the engine.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-ctx", type=int, default=131072)
    ap.add_argument("--groups-used", type=int, default=8)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--ef", type=int, default=128)
    a = ap.parse_args()
    import torch
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    spec = WorkloadSpec(n_ctx=a.n_ctx, d_model=256, d_head=128, n_heads=32, n_kv_groups=8,
                        seed=7, n_decode=a.steps + 1)
    kvs, graphs, dq = [], [], []
    bp = ra.OODGraphBuildParams(128, 24, 256, 8)
    for g in range(a.groups_used):
        w = generate_group(spec, g, "cuda")
        kv = ra.KVGroup(w["keys"], w["values"])
        kvs.append(kv)
        for m in range(4):
            graphs.append(ra.ood_build(kv, w["prefill_q"][m], bp))
            dq.append(w["decode_q"][m])
    Q = torch.stack(dq, dim=1).contiguous()
    eng = ra.Engine(kvs, graphs, ra.EngineConfig(128, 512, 100, a.ef))
    for i in range(a.steps):
        eng.decode_step_device(Q[i])
    torch.cuda.synchronize()
    s, e = eng.last_stats()
    print(f"steps={a.steps} heads={len(graphs)} scanned/head={s / len(graphs):.1f} "
          f"expanded/head={e / len(graphs):.1f} timing={eng.last_timing()}")
    dc = eng.debug_counters()
    print({k: v / len(graphs) for k, v in dc.items()})


if __name__ == "__main__":
    main()
