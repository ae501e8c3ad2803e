#!/usr/bin/env python3
"""Decode-attention benchmark: RetrievalAttention hot path at Llama-3-8B shape.

Workload (BASELINE.json configs[1]): one layer, 32 query heads over 8 KV
groups, d_head 128, 128K context, static set = first 128 + last 512 tokens,
top-100 retrieval per head through the head's OODGraph (k_train 128, M 24,
efc 256, window 8; README/acceptance parameters), ef 128. Inputs are the
reference generator's synthetic OOD K/Q/V (seed 7), synthesized on the GPU
(paper_2409_10516_b200.workload); graphs are built on the GPU (untimed).

One step = ra_engine decode step for all local heads: graph search ->
partial attention over W -> partial over Omega -> LSE merge (+ NCCL
all_gather of per-head outputs when N > 1, heads sharded by KV group).
Metric: ms per decode step (token) for the layer, lower is better.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attention ms/token @128K (Llama-3-8B shape); search recall@100; HBM GB/s"
TPUT_R = 128  # batched line: 128 decode queries per head x 32 heads = 4096 searches


def workload_config(a, H, G):
    """The workload both arms run (BASELINE.json configs[1])."""
    return {"workload": "configs[1]: Llama-3-8B shape single layer, 32 Q heads / 8 KV "
                        "groups, d=128, 128K ctx, top-100 + 640 static, ef 128",
            "n_ctx": a.n_ctx, "heads": H, "kv_groups": G, "top_k": a.top_k, "ef": a.ef,
            "graph": {"k_train": a.k_train, "max_degree": a.max_degree,
                      "ef_construction": a.ef_construction, "edge_window": 8},
            "l2": f"flushed between timed steps ({a.flush_mb} MiB write)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-ctx", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--ef", type=int, default=128)
    ap.add_argument("--top-k", type=int, default=100)
    ap.add_argument("--k-train", type=int, default=128)
    ap.add_argument("--max-degree", type=int, default=24)
    ap.add_argument("--ef-construction", type=int, default=256)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-bf16", action="store_true", help="skip the bf16-KV measurement")
    ap.add_argument("--no-throughput", action="store_true",
                    help="skip the batched (throughput-mode) line (launch-list profiling)")
    ap.add_argument("--no-multilayer", action="store_true",
                    help="skip the 4-distinct-layer batched measurement")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--shard", default="layers", choices=["layers", "heads"],
                    help="N>1: layers = weak scaling, rank r decodes its own synthetic layer "
                         "(seed 7 + r, all 32 heads, no data-path collective); heads = strong "
                         "scaling, the layer's KV groups split over ranks + NCCL all_gather "
                         "of per-head outputs")
    return ap.parse_args()


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML
    (pynvml, ~1 ms per sample) when available, else nvidia-smi polling."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.stop = device, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.bits = (pynvml.nvmlClocksEventReasonHwSlowdown,
                         pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwPowerCap)
        except Exception:
            self.nvml = None

    def sample(self):
        if self.nvml is not None:
            p = self.nvml
            sm = p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM)
            r = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            return [sm, self.max_mhz] + [bool(r & b) for b in self.bits]
        out = subprocess.run(
            ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits"], capture_output=True, text=True,
            timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        return [float(f[0]), float(f[1])] + [x.lower().startswith("active") for x in f[2:6]]

    def run(self):
        while not self.stop.is_set():
            try:
                self.rows.append(self.sample())
            except Exception:
                pass
            self.stop.wait(0.004 if self.nvml is not None else 0.2)

    def __enter__(self):
        # the sampler thread must not hold the GIL across the main thread's
        # launches for long: a short switch interval bounds that wait
        self.switch = sys.getswitchinterval()
        sys.setswitchinterval(0.0002)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)
        sys.setswitchinterval(self.switch)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def measured_peaks():
    """HBM GB/s from the driver-written MEASURED_PEAKS.json (any numeric entry
    whose key path names HBM bandwidth; TB/s values are scaled), else the
    profiling recipe's 6650 GB/s fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except Exception:
        return 6650.0, "fallback"
    found = []

    def walk(node, path):
        if isinstance(node, dict):
            for k, v in node.items():
                walk(v, path + [str(k).lower()])
        elif isinstance(node, (int, float)) and not isinstance(node, bool):
            key = "/".join(path)
            if "hbm" in key and not any(t in key for t in ("tflop", "pflop", "clock", "mhz")):
                found.append((key, float(node)))

    walk(p, [])
    for key, v in sorted(found, key=lambda kv: ("copy" not in kv[0] and "gb" not in kv[0],
                                                 kv[0])):
        gbs = v * 1000.0 if v < 100 else v  # a TB/s figure
        if 1000.0 < gbs < 20000.0:
            return gbs, "measured"
    return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of the search kernel from the committed ncu
    --set full capture (profiles/ncu_search_summary.json), if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_search_summary.json")) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference" and rank != 0:
        return  # the reference CPU arm runs on rank 0 only
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1 and a.impl == "ours":
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group

    H, G = a.heads, a.groups
    hpg = H // G
    n_world = world if a.impl == "ours" else 1
    from paper_2409_10516_b200.shard import OutputGather, groups_for_rank
    by_heads = a.shard == "heads" and n_world > 1
    my_groups = (groups_for_rank(G, n_world, rank) if by_heads else list(range(G)))
    layer = rank if (a.impl == "ours" and not by_heads) else 0
    # decode queries: the timed steps, the e2e steps, and one batched step of
    # TPUT_R queries per head (the throughput line)
    n_dec = max(a.warmup + 2 * a.steps + 2, TPUT_R)
    # synthetic layer l uses seed 7 + l (SURVEY §8 d; the reference has no layers)
    spec = WorkloadSpec(n_ctx=a.n_ctx, d_model=256, d_head=128, n_heads=H, n_kv_groups=G,
                        seed=7 + layer, n_decode=n_dec)
    dev = torch.device("cuda", local)
    t0 = time.time()
    kvs, graphs, dq, keys_host, vals_host = [], [], [], [], []
    bp = ra.OODGraphBuildParams(a.k_train, a.max_degree, a.ef_construction, 8)
    build_ms = []
    for g in my_groups:
        w = generate_group(spec, g, dev)
        kv = ra.KVGroup(w["keys"], w["values"])
        kvs.append(kv)
        for m in range(hpg):
            torch.cuda.synchronize()
            tb = time.time()
            graphs.append(ra.ood_build(kv, w["prefill_q"][m], bp))
            build_ms.append((time.time() - tb) * 1e3)
            dq.append(w["decode_q"][m])
        if a.impl == "reference" or rank == 0:
            keys_host.append(w["keys"].cpu().numpy())
            vals_host.append(w["values"].cpu().numpy())
        del w
    setup_s = time.time() - t0
    Hl = len(graphs)
    Q = torch.stack(dq, dim=1).contiguous()  # [n_dec, Hl, d]: Q[i] is one step, contiguous
    del dq
    cfg = ra.EngineConfig(128, 512, a.top_k, a.ef)

    if a.impl == "reference":
        run_reference(a, keys_host, vals_host, graphs, Q, cfg, H, G, setup_s)
        return

    eng = ra.Engine(kvs, graphs, cfg)
    stream = torch.cuda.current_stream()
    flush = torch.empty(a.flush_mb * (1 << 20) // 4, dtype=torch.float32, device=dev)
    gather = OutputGather(G, hpg, 128, world, rank, dev) if (dist is not None and by_heads) else None

    def step(i):
        out, om, sc = eng.decode_step_device(Q[i])
        if gather is not None:
            gather(out, dist)  # all heads' outputs on every rank (NCCL all_gather)
        return out

    for i in range(a.warmup):
        step(i)
    eng.last_timing(), eng.last_stats()  # first-call paths outside the timed loop
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    times, search_ms, attn_ms, scanned, expanded = [], [], [], [], []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(a.warmup, a.warmup + a.steps):
            flush.zero_()  # evict L2 between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(i)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            s_ms, a_ms = eng.last_timing()
            search_ms.append(s_ms)
            attn_ms.append(a_ms)
            s, e = eng.last_stats()
            scanned.append(s)
            expanded.append(e)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()

    # ---- end-to-end through the host API (H2D q, D2H out/omega/scanned) ----
    qh = torch.empty((Hl, 128), dtype=torch.float32, pin_memory=True)
    out_h = torch.empty((Hl, 128), dtype=torch.float64, pin_memory=True)
    om_h = torch.empty((Hl, max(eng.k, 1)), dtype=torch.int32, pin_memory=True)
    sc_h = torch.empty(Hl, dtype=torch.int64, pin_memory=True)
    Qh = Q.cpu()
    e2e = []
    for i in range(a.warmup + a.steps, a.warmup + 2 * a.steps):
        qh.copy_(Qh[i])
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.ctx.bind_stream()
        ra.api._check(ra.lib.ra_engine_step_host(eng.h, qh.data_ptr(), out_h.data_ptr(),
                                                 om_h.data_ptr(), sc_h.data_ptr()))
        e1.record(stream)
        e1.synchronize()
        e2e.append(e0.elapsed_time(e1))

    tput = (batched_throughput(a, ra, kvs, graphs, Q, cfg, flush, stream)
            if not a.no_throughput else None)
    tput_ml = (multilayer_throughput(a, ra, spec, my_groups, hpg, kvs, graphs, Q, cfg, flush,
                                     stream, layer) if not a.no_multilayer else None)
    out32 = eng.decode_step_device(Q[a.warmup])[0].cpu().numpy()
    bf16 = (bf16_mode(a, ra, spec, my_groups, hpg, Q, cfg, flush, stream, out32, graphs)
            if not a.no_bf16 else None)

    ms = statistics.mean(times)
    ms_search = statistics.mean(search_ms)
    ms_e2e = statistics.mean(e2e)
    if dist is not None:
        t = torch.tensor([ms, ms_e2e, ms_search], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e, ms_search = (float(x) for x in t)
        # shard balance: per-rank mean scanned per head, max vs mean
        sc_local = torch.tensor([statistics.mean(scanned) / max(Hl, 1)], dtype=torch.float64,
                                device=dev)
        all_sc = [torch.zeros_like(sc_local) for _ in range(world)]
        dist.all_gather(all_sc, sc_local)
        per_rank = [float(x) for x in all_sc]
        shard_balance = {"mean_scanned_per_head_by_rank": [round(x, 1) for x in per_rank],
                         "max_over_mean": round(max(per_rank) / statistics.mean(per_rank), 4)}
    else:
        shard_balance = None
    # whole-job aggregate: layer-sharded ranks each decode one layer per step,
    # so N layer-tokens complete in the (max-over-ranks) step time
    units = world if (dist is not None and not by_heads) else 1
    step_ms, ms, ms_e2e = ms, ms / units, ms_e2e / units
    d, M = 128, a.max_degree
    bytes_search = statistics.mean([s * d * 4 + e * M * 4 + 0.0 for s, e in zip(scanned, expanded)])
    fused = eng.kernels_per_step() == 1
    if fused:  # the kernel also reads W's K and V rows (once per group) and the Omega V rows
        nW = min(128, a.n_ctx) + min(512, max(a.n_ctx - 128, 0))
        bytes_search += len(my_groups) * nW * d * 8 + Hl * a.top_k * d * 4
    peak, peak_kind = measured_peaks()
    achieved = bytes_search / (statistics.mean(search_ms) * 1e-3) / 1e9
    res = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms/token", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(step_ms, 4),
        "higher_is_better": False, "scaling": "strong" if by_heads else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference OOD generator algorithm, seed 7, GPU-synthesized)",
        "config": dict(workload_config(a, H, G),
                       parallelism=(f"heads sharded by KV group over {world} GPU(s) + NCCL "
                                    "all_gather of outputs" if by_heads else
                                    f"layer-sharded: {world} GPU(s), rank r decodes synthetic "
                                    "layer r (all 32 heads), no data-path collective; value = "
                                    "step time / layers")),
        "e2e": {"value": round(ms_e2e, 4), "unit": "ms/token",
                "h2d_bytes_per_step": Hl * 128 * 4,
                "d2h_bytes_per_step": Hl * 128 * 8 + Hl * max(eng.k, 1) * 4 + Hl * 8},
        # fused step: 1 kernel (search + W / Omega partials + merge), else 3
        "gpu_launches": eng.kernels_per_step() * a.steps,
        "roofline": {"bound": "hbm",
                     "kernel": "k_graph_search_pipe (latency mode" +
                               (", fused attention: search + W / Omega partials + merge)"
                                if fused else ")"),
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 5), "peak_source": peak_kind,
                     "traffic": ncu_traffic(),
                     "algorithmic_bytes_per_launch": int(bytes_search),
                     "search_ms": round(ms_search, 4),
                     "attention_ms": round(statistics.mean(attn_ms), 4)},
        "search": {"mean_scanned_per_head": statistics.mean(scanned) / Hl,
                   "mean_expanded_per_head": statistics.mean(expanded) / Hl,
                   "scan_fraction": statistics.mean(scanned) / Hl / (a.n_ctx - 640)},
        "clocks": clk.summary(),
        "throughput": tput,
        "throughput_multilayer": tput_ml,
        "shard_balance": shard_balance,
        "bf16_kv": bf16,
        "setup_s": round(setup_s, 1),
        "build_ms_per_head": round(statistics.mean(build_ms), 1),
        "build_phase_ms_per_head": {
            k: round(statistics.mean(g.build_stats.ms[k] for g in graphs), 2)
            for k in ("knn", "knn_tensor", "edges", "prune", "entry", "repair")},
        "build_knn_rows_exact_fallback": sum(g.build_stats.knn_rows_widened for g in graphs),
    }
    if rank == 0:
        res["recall"] = recall(eng, graphs, kvs, Q, a, ra)
        if world == 1 and not a.no_cpu_baseline:
            res["cpu_baseline"], res["parity"] = cpu_baseline(a, keys_host, vals_host, graphs,
                                                              Q, cfg, eng)
        print(json.dumps(res))
    if dist is not None:
        dist.destroy_process_group()


def batched_throughput(a, ra, kvs, graphs, Q, cfg, flush, stream, row_bytes=512):
    """Batched decode: R decode queries per head issued as ONE engine step
    over R x H heads (graphs and KV groups repeated R times, so every query
    walks its head's real graph and KV): search (throughput-mode kernel) +
    static/retrieved partial attention + merge for R x H queries (R = 128:
    4096 searches, the per-GPU search count of configs[2] - 32 layers x batch
    8 - sharded over 2 GPUs) with the layer's KV shared by the R queries of a
    head."""
    import torch
    R = min(TPUT_R, Q.shape[0])
    Hl = len(graphs)
    eng = ra.Engine(list(kvs) * R, list(graphs) * R, cfg)
    qb = [Q[j:j + R].reshape(R * Hl, -1).contiguous()
          for j in range(0, Q.shape[0] - R + 1, R)]
    for i in range(3):
        eng.decode_step_device(qb[i % len(qb)])
    torch.cuda.synchronize()
    times, s_ms, sc, ex = [], [], [], []
    for i in range(max(3, min(a.steps, 10))):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.decode_step_device(qb[i % len(qb)])
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        s_ms.append(eng.last_timing()[0])
        s, e = eng.last_stats()
        sc.append(s)
        ex.append(e)
    ms, ms_s = statistics.mean(times), statistics.mean(s_ms)
    by = statistics.mean([s * row_bytes + e * a.max_degree * 4 for s, e in zip(sc, ex)])
    peak, kind = measured_peaks()
    gbs = by / (ms_s * 1e-3) / 1e9
    del eng
    return {"queries_per_step": R * Hl, "decode_queries_per_head": R,
            "ms_per_step": round(ms, 4), "us_per_query": round(ms * 1e3 / (R * Hl), 3),
            "queries_per_s": round(R * Hl / (ms * 1e-3), 1),
            "search_ms": round(ms_s, 4), "search_kernel": "k_graph_search_pipe (TP mode)",
            "search_algorithmic_bytes": int(by),
            "search_GBps": round(gbs, 1), "search_frac": round(gbs / peak, 4),
            "peak_source": kind,
            "note": "one engine step over R x H heads; KV of each head shared by its R queries"}


def multilayer_throughput(a, ra, spec, my_groups, hpg, kvs0, graphs0, Q0, cfg, flush, stream,
                          layer0, n_layers=4, R=32):
    """Layer-batched decode with DISTINCT layers: this layer plus 3 more
    synthetic layers (seeds 7 + l, their own K/V and graphs), 32 decode
    queries per head per layer, all 4096 searches + attention in one engine
    step (configs[2]'s per-GPU shape with 4 layers x batch 32)."""
    import dataclasses
    import torch
    from paper_2409_10516_b200.workload import generate_group
    bp = ra.OODGraphBuildParams(a.k_train, a.max_degree, a.ef_construction, 8)
    layers = [(list(kvs0), list(graphs0), Q0[:R])]
    for l in range(1, n_layers):
        sp = dataclasses.replace(spec, seed=7 + layer0 * n_layers + l, n_decode=R)
        kvs, graphs, dq = [], [], []
        for g in my_groups:
            w = generate_group(sp, g, Q0.device)
            kv = ra.KVGroup(w["keys"], w["values"])
            kvs.append(kv)
            for m in range(hpg):
                graphs.append(ra.ood_build(kv, w["prefill_q"][m], bp))
                dq.append(w["decode_q"][m])
            del w
        layers.append((kvs, graphs, torch.stack(dq, dim=1)))
    G_all = [kv for kvs, _, _ in layers for _ in range(R) for kv in kvs]
    H_all = [g for _, gr, _ in layers for _ in range(R) for g in gr]
    eng = ra.Engine(G_all, H_all, cfg)
    q = torch.cat([dq[:R].reshape(R * dq.shape[1], -1) for _, _, dq in layers]).contiguous()
    for _ in range(3):
        eng.decode_step_device(q)
    torch.cuda.synchronize()
    times, s_ms, sc, ex = [], [], [], []
    for _ in range(max(3, min(a.steps, 10))):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.decode_step_device(q)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        s_ms.append(eng.last_timing()[0])
        s, e = eng.last_stats()
        sc.append(s)
        ex.append(e)
    ms, ms_s = statistics.mean(times), statistics.mean(s_ms)
    nq = len(H_all)
    by = statistics.mean([s * 512 + e * a.max_degree * 4 for s, e in zip(sc, ex)])
    peak, kind = measured_peaks()
    gbs = by / (ms_s * 1e-3) / 1e9
    del eng
    return {"layers": n_layers, "decode_queries_per_head_per_layer": R, "queries_per_step": nq,
            "ms_per_step": round(ms, 4), "us_per_query": round(ms * 1e3 / nq, 3),
            "queries_per_s": round(nq / (ms * 1e-3), 1), "search_ms": round(ms_s, 4),
            "search_GBps": round(gbs, 1), "search_frac": round(gbs / peak, 4),
            "peak_source": kind,
            "note": "distinct synthetic layers (own K/V and graphs); one engine step"}


def bf16_mode(a, ra, spec, my_groups, hpg, Q, cfg, flush, stream, out32, graphs32):
    """The same decode step on bf16 KV groups, two ways:
    bf16      - K/V rounded to bf16 (nearest even), graphs rebuilt on the
                rounded keys from the same prefill queries: exactly the
                reference's results on the rounded inputs, half the bytes;
    bf16_attn - the search keeps the exact f32 keys (ids identical to f32,
                graphs reused), the sparse attention reads bf16 K/V.
    Per mode: step time, the batched line, the output's distance from f32."""
    import torch
    from paper_2409_10516_b200.workload import generate_group
    bp = ra.OODGraphBuildParams(a.k_train, a.max_degree, a.ef_construction, 8)
    res = {}
    for mode in ("bf16", "bf16_attn"):
        kvs, graphs = [], []
        for gi, g in enumerate(my_groups):
            w = generate_group(spec, g, Q.device)
            kv = ra.KVGroup(w["keys"], w["values"], dtype=mode)
            kvs.append(kv)
            if mode == "bf16":
                graphs += [ra.ood_build(kv, w["prefill_q"][m], bp) for m in range(hpg)]
            else:
                graphs += [ra.OODGraph.from_blob(kv, graphs32[gi * hpg + m].serialize())
                           for m in range(hpg)]
            del w
        eng = ra.Engine(kvs, graphs, cfg)
        for i in range(a.warmup):
            eng.decode_step_device(Q[i])
        torch.cuda.synchronize()
        times, s_ms, sc, ex = [], [], [], []
        for i in range(a.warmup, a.warmup + a.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.decode_step_device(Q[i])
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            s_ms.append(eng.last_timing()[0])
            s, e = eng.last_stats()
            sc.append(s)
            ex.append(e)
        o = eng.decode_step_device(Q[a.warmup])[0].cpu().numpy()
        rel = np.linalg.norm(o - out32, axis=1) / np.linalg.norm(out32, axis=1)
        rb = 256 if mode == "bf16" else 512
        by = statistics.mean([s_ * rb + e_ * a.max_degree * 4 for s_, e_ in zip(sc, ex)])
        tput = batched_throughput(a, ra, kvs, graphs, Q, cfg, flush, stream, row_bytes=rb)
        del eng
        res[mode] = {"value": round(statistics.mean(times), 4), "unit": "ms/token",
                     "search_ms": round(statistics.mean(s_ms), 4),
                     "search_GBps": round(by / (statistics.mean(s_ms) * 1e-3) / 1e9, 1),
                     "out_rel_vs_f32": {"max": float(rel.max()), "mean": float(rel.mean())},
                     "throughput_us_per_query": tput["us_per_query"],
                     "throughput_search_GBps": tput["search_GBps"]}
    res["note"] = ("bf16: K/V rounded in HBM, graphs rebuilt on the rounded keys (= the "
                   "reference on the rounded inputs); bf16_attn: exact f32 search (same ids), "
                   "bf16 K/V in the attention; north-star bf16 tolerance 1e-2")
    return res


def recall(eng, graphs, kvs, Q, a, ra):
    """recall@100 on a sample against the GPU FlatIndex (exact, the
    reference's recall ground truth, index_flat.hpp:9-22): engine-level
    (masked by W, vs the exact pool top-100, acceptance.cpp:207-212) and
    unmasked graph search vs FlatIndex (diagnostics.cpp:150-164)."""
    hpg = a.heads // a.groups
    W = ra.static_partition(a.n_ctx, 128, 512).static_set
    flats = [ra.FlatIndex(kv) for kv in kvs]
    rec_m, rec_u = [], []
    for i in range(min(4, a.steps)):
        q = Q[a.warmup + i]
        out, om, sc = eng.decode_step_device(q)
        omega = om.cpu().numpy().view(np.uint32)
        un = ra.search_batch(graphs, q, 100, None, a.ef).host()
        for g, flat in enumerate(flats):
            qg = q[g * hpg:(g + 1) * hpg]
            tm = flat.search_batch(qg, 100, W)
            tu = flat.search_batch(qg, 100)
            for j in range(hpg):
                h = g * hpg + j
                rec_m.append(len(set(tm[j].ids.tolist()) & set(omega[h].tolist())) / 100)
                rec_u.append(len(set(tu[j].ids.tolist()) & set(un[h].ids.tolist())) / 100)
    return {"masked_engine": round(float(np.mean(rec_m)), 4),
            "unmasked_flat": round(float(np.mean(rec_u)), 4), "samples": len(rec_m),
            "ef": a.ef, "ground_truth": "ra_flat_search_batch (GPU FlatIndex)"}


def _ref_engine(keys_host, vals_host, graphs, cfg, threads):
    from oracle.ffi import Oracle, available
    if not available("ref"):
        return None, None
    o = Oracle("ref")
    blobs = [g.serialize() for g in graphs]
    eng = o.engine(np.stack(keys_host), np.stack(vals_host), blobs, cfg.s_init, cfg.s_local,
                   cfg.top_k, cfg.search_param, threads)
    return o, eng


def cpu_baseline(a, keys_host, vals_host, graphs, Q, cfg, eng):
    """The reference's own decode_step (oracle/_ref, unmodified sources) on the
    host cores over the same graphs (loaded through OODGraph(keys, blob)),
    bounded to ~cpu_seconds; doubles as a full-size parity check."""
    threads = os.cpu_count() or 1
    o, reng = _ref_engine(keys_host, vals_host, graphs, cfg, threads)
    if reng is None:
        return {"value": None, "unavailable": "oracle/_ref not built"}, None
    Qh = Q.cpu().numpy()
    times, same_om, same_sc, max_rel, n = [], 0, 0, 0.0, 0
    t_end = time.time() + a.cpu_seconds
    i = a.warmup
    while (time.time() < t_end or not times) and i < Q.shape[0]:
        q = np.ascontiguousarray(Qh[i])
        t0 = time.perf_counter()
        rout, rom, rsc = reng.step(q, i)
        times.append((time.perf_counter() - t0) * 1e3)
        if not a.no_parity:
            out, om, sc = eng.decode_step(q)
            same_om += int((om == rom[:, : om.shape[1]]).all(axis=1).sum())
            same_sc += int((sc == rsc).sum())
            rel = np.linalg.norm(out - rout, axis=1) / np.linalg.norm(rout, axis=1)
            max_rel = max(max_rel, float(rel.max()))
            n += q.shape[0]
        i += 1
    base = {"value": round(statistics.mean(times), 3), "unit": "ms/token", "cores": threads,
            "kind": "reference",
            "sample": f"{len(times)} decode steps x {Qh.shape[1]} heads at n_ctx {a.n_ctx} "
                      f"(reference decode_step, n_threads={threads}, GPU-built graphs via OODG)"}
    parity = None if a.no_parity else {
        "heads_checked": n, "omega_identical": same_om, "scanned_identical": same_sc,
        "max_out_rel_err": max_rel}
    return base, parity


def run_reference(a, keys_host, vals_host, graphs, Q, cfg, H, G, setup_s):
    threads = os.cpu_count() or 1
    o, reng = _ref_engine(keys_host, vals_host, graphs, cfg, threads)
    if reng is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    Qh = Q.cpu().numpy()
    for i in range(a.warmup):
        reng.step(np.ascontiguousarray(Qh[i]), i)
    times = []
    t_start = time.perf_counter()
    for i in range(a.warmup, a.warmup + a.steps):
        t0 = time.perf_counter()
        reng.step(np.ascontiguousarray(Qh[i]), i)
        times.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.mean(times)
    sample = (f"{a.steps} reference decode_steps x {H} heads at n_ctx {a.n_ctx} "
              f"(n_threads={threads}; graphs built on GPU, loaded via OODG blobs)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(ms, 3), "unit": "ms/token",
        "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference OOD generator algorithm, seed 7)",
        "config": dict(workload_config(a, H, G),
                       parallelism="reference decode_step on the host cores (rank 0)"),
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/token", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(ms, 3), "unit": "ms/token", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_start, 2), "setup_s": round(setup_s, 1)}))


if __name__ == "__main__":
    main()
