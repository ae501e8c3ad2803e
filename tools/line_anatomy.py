#!/usr/bin/env python3
"""Per-search anatomy of the multi-context (layers32-shaped) step
(profiling aid): for each K6 variant, the CUDA-event search time and, per
search, clock64 cycles, expansions and the throughput-mode overflow
counters (FO/UO spill rounds, FO pops, moved-to-HBM flags).

  python tools/line_anatomy.py --layers 32 --kernels tps,tp
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-ctx", type=int, default=131072)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--kernels", default="tps,tp")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "line_anatomy.json"))
    a = ap.parse_args()
    import torch
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    bp = ra.OODGraphBuildParams(128, 24, 256, 8)
    kvs, graphs, dq = [], [], []
    t0 = time.time()
    for l in range(a.layers):
        spec = WorkloadSpec(n_ctx=a.n_ctx, d_model=256, d_head=128, n_heads=32,
                            n_kv_groups=8, seed=7 + l, n_decode=a.steps + 1)
        for g in range(a.groups):
            w = generate_group(spec, g, "cuda")
            kv = ra.KVGroup(w["keys"], w["values"])
            kvs.append(kv)
            for m in range(4):
                graphs.append(ra.ood_build(kv, w["prefill_q"][m], bp))
                dq.append(w["decode_q"][m])
            del w
    print(f"setup {time.time() - t0:.1f} s, {len(graphs)} heads", flush=True)
    Q = torch.stack(dq, dim=1).contiguous()
    flush = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
    ctx = ra.default_context()
    report = {}
    for kern in a.kernels.split(","):
        ctx.set_search_kernel(kern)
        eng = ra.Engine(kvs, graphs, ra.EngineConfig(128, 512, 100, 128))
        eng.decode_step_device(Q[0])
        ms = []
        cs = []
        for i in range(a.steps):
            flush.zero_()
            torch.cuda.synchronize()
            eng.decode_step_device(Q[i])
            ms.append(eng.last_timing()[0])
            cs.append(eng.debug_counters_per_head().astype(np.float64))
        c = np.concatenate(cs)  # every (step, head)
        cyc, exp = c[:, 2], c[:, 3]
        r = {"search_ms": ms, "kernels_per_step": eng.kernels_per_step(),
             "cycles_mean": float(cyc.mean()), "cycles_p50": float(np.median(cyc)),
             "cycles_p99": float(np.percentile(cyc, 99)), "cycles_max": float(cyc.max()),
             "expanded_mean": float(exp.mean()), "expanded_max": float(exp.max()),
             "cycles_per_expansion_mean": float((cyc / np.maximum(exp, 1)).mean()),
             "corr_cycles_expanded": float(np.corrcoef(cyc, exp)[0, 1]),
             "fo_spill_rounds_mean": float(c[:, 7].mean()), "fo_pops_mean": float(c[:, 8].mean()),
             "fo_to_hbm": int((c[:, 9].astype(int) & 1).sum()),
             "uo_to_hbm": int((c[:, 9].astype(int) & 2).sum()),
             "uo_spill_rounds_mean": float(c[:, 10].mean()),
             "peak_FO_p99": float(np.percentile(c[:, 5], 99)), "peak_FO_max": float(c[:, 5].max()),
             "peak_UO_p99": float(np.percentile(c[:, 11], 99)), "peak_UO_max": float(c[:, 11].max()),
             "compactions_mean": float(c[:, 6].mean()),
             "misses_mean": float(c[:, 0].mean()),
             # duo: the commit warp's packet waits / the expansion warp's busy cycles
             "wait_cycles_mean": float(c[:, 1].mean()),
             "dbg_slot_means": [float(c[:, j].mean()) for j in range(12)],
             "hit_or_helper_busy_cycles_mean": float(c[:, 4].mean()),
             # RA_PIPE_PROFILE builds: per-phase cycles (top/stop, pop, expand, visit)
             "profile_cycles_mean": [float(c[:, j].mean()) for j in (7, 8, 9, 10)],
             "profile_adj_tma_cycles_mean": [float(c[:, 5].mean()), float(c[:, 11].mean())]}
        slow = np.argsort(-cyc)[:8]
        r["slowest"] = [{"head": int(h), "cycles": float(cyc[h]), "expanded": float(exp[h]),
                         "fo_pops": float(c[h, 8]), "fo_flags": int(c[h, 9])} for h in slow]
        report[kern] = r
        print(kern, json.dumps({k: v for k, v in r.items() if k != "slowest"}), flush=True)
        del eng
    ctx.set_search_kernel(None)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
