#!/usr/bin/env python3
"""Profiling driver: one GPU graph build at --n keys / queries (d=128).
  ncu --set full -k regex:k_knn_tc -c 1 -o gpurun_out/knn python tools/profile_build.py --n 32768
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--heads", type=int, default=1, help="distinct prefill-query sets (of 4)")
    ap.add_argument("--group", type=int, default=0, help="KV group of the 8-group workload")
    a = ap.parse_args()
    import torch
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    w = generate_group(WorkloadSpec(n_ctx=a.n, d_model=256, d_head=128, n_heads=32, n_kv_groups=8,
                                    seed=7, n_decode=1), a.group, "cuda")
    kv = ra.KVGroup(w["keys"], w["values"])
    torch.cuda.synchronize()
    for r in range(a.reps):
        t = time.time()
        g = ra.ood_build(kv, w["prefill_q"][r % a.heads], ra.OODGraphBuildParams(128, 24, 256, 8))
        ms = {k: round(v, 1) for k, v in g.build_stats.ms.items()}
        print(f"n={a.n} build {1e3 * (time.time() - t):.1f} ms phases {ms} "
              f"repair rounds {g.build_stats.repair_rounds} nodes {g.build_stats.repaired_nodes} "
              f"fallback_rows {g.build_stats.knn_rows_widened}")


if __name__ == "__main__":
    main()
