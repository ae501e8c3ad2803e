#!/usr/bin/env python3
"""Per-head anatomy of the search kernel at config 2 (profiling aid):
rounds, expansions, scanned and clock64 cycles per phase for every head,
plus the CUDA-event search time. Same workload as bench.py."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-ctx", type=int, default=131072)
    ap.add_argument("--groups-used", type=int, default=8)
    ap.add_argument("--steps", type=int, default=6)
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
    flush = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
    tot = []
    for i in range(a.steps):
        flush.zero_()
        eng.decode_step_device(Q[i])
        torch.cuda.synchronize()
        s_ms, _ = eng.last_timing()
        d = eng.debug_counters_per_head().astype(np.float64)
        sc = eng.scanned.cpu().numpy()
        if i >= 2:
            tot.append((s_ms, d, sc))
    s_ms, d, sc = tot[-1]
    clk = 1.965e3  # cycles per us at max SM clock
    print(f"search_ms per step: {[round(t[0], 4) for t in tot]}")
    if os.environ.get("RA_SEARCH_KERNEL", "pipe") == "pipe":
        cols = ["miss", "wait_us", "total_us", "commits", "hits", "helper_exp", "compactions",
                "top_us", "pop_us", "lookup_us", "visit_us", "compact_us"]
        print("head scanned " + " ".join(cols))
        for h in range(d.shape[0]):
            r = d[h].copy()
            r[1] /= clk
            r[2] /= clk
            r[7:] /= clk
            print(f"{h:3d} {int(sc[h]):6d} " + " ".join(f"{x:9.1f}" for x in r))
        if os.environ.get("RA_MISSCLASS"):
            raw = d[:, 9].astype(np.uint64)
            coll, empty, own = raw & 0xFFFFF, (raw >> 20) & 0xFFFFF, raw >> 40
            print(f"miss classes (mean/head): child of a packet {coll.mean():.1f} "
                  f"child of an inline expansion {empty.mean():.1f} older {own.mean():.1f}")
        print("mean  " + " ".join(f"{c}={d[:, j].mean() / (clk if j in (1, 2, 7, 8, 9, 10, 11) else 1):.1f}"
                                  for j, c in enumerate(cols)))
        return
    print("head rounds commits scanned cyc_pre(us) cyc_commit(us) argmax stop packet add select")
    for h in range(d.shape[0]):
        r = d[h]
        print(f"{h:3d} {int(r[0]):5d} {int(r[3]):5d} {int(sc[h]):6d} {r[1]/clk:9.1f} {r[2]/clk:9.1f} "
              + " ".join(f"{r[4 + j]/clk:7.1f}" for j in range(5)))
    mx = int(np.argmax(d[:, 1] + d[:, 2]))
    r = d[mx]
    print(f"slowest head {mx}: rounds {int(r[0])}, commits {int(r[3])}, "
          f"us/round pre {r[1]/clk/r[0]:.2f} commit {r[2]/clk/r[0]:.2f}")
    print(f"mean: rounds {d[:,0].mean():.1f} commits {d[:,3].mean():.1f} "
          f"commits/round {(d[:,3]/d[:,0]).mean():.2f}")


if __name__ == "__main__":
    main()
