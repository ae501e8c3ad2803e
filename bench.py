#!/usr/bin/env python3
"""Decode-attention benchmark: RetrievalAttention hot path at Llama-3-8B shape.

Headline workload (BASELINE.json configs[1]): one layer, 32 query heads over
8 KV groups, d_head 128, 128K context, static set = first 128 + last 512
tokens, top-100 retrieval per head through the head's OODGraph (k_train
128, M 24, efc 256, window 8; README/acceptance parameters), ef 128. Inputs
are the reference generator's synthetic OOD K/Q/V (seed 7), synthesized on
the GPU (paper_2409_10516_b200.workload, equal to the reference generator's
output: tests/test_workload_gpu.py); graphs are built on the GPU (untimed).

One step = ra_engine decode step for all local heads: graph search ->
partial attention over W -> partial over Omega -> LSE merge.
Metric: ms per decode step (token) for the layer, lower is better.

Further lines in the same JSON object (`lines`), each with its own
roofline: `layers32` (the north-star shape: 32 distinct layers x 8 KV
groups x 4 heads at 128K, batch 1, one token = 1024 searches + attention),
`batch8` (configs[2]'s per-GPU shard at 8 GPUs: 32 layers x 1 KV group x 8
distinct batch contexts), `ctx_1m` (configs[4]: one full layer at a 1M-token
context on one GPU).

`--impl reference` runs the reference's own CPU path end to end from
oracle/_ref (unmodified reference sources): generate_workload +
engine_init (OODGraph builds) + decode_step, on the host cores, with no
code of this repo on its path.

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


def workload_config(a, H, G):
    """The workload both arms run (BASELINE.json configs[1]); identical dicts
    in both arms (how each arm executes goes to the line's `execution`)."""
    return {"workload": "configs[1]: Llama-3-8B shape single layer, 32 Q heads / 8 KV "
                        "groups, d=128, 128K ctx, top-100 + 640 static, ef 128",
            "n_ctx": a.n_ctx, "heads": H, "kv_groups": G, "top_k": a.top_k, "ef": a.ef,
            "graph": {"k_train": a.k_train, "max_degree": a.max_degree,
                      "ef_construction": a.ef_construction, "edge_window": 8},
            "seed": 7,
            "parallelism": (f"{a.gpus} GPU(s), " + ("KV groups sharded over ranks + NCCL "
                                                    "all_gather of outputs"
                                                    if a.shard == "heads" else
                                                    "rank r decodes synthetic layer r")
                            if a.gpus > 1 else "single device"),
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
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--no-layers32", action="store_true",
                    help="skip the 32-distinct-layer line (north-star shape)")
    ap.add_argument("--no-batch8", action="store_true",
                    help="skip configs[2]'s per-GPU shard line (32 layers x batch 8)")
    ap.add_argument("--no-1m", action="store_true", help="skip the 1M-context line")
    ap.add_argument("--lines-only", default="",
                    help="comma list of lines to run (layers32,batch8,ctx_1m); "
                         "skips the headline measurement (profiling)")
    ap.add_argument("--line-layers", type=int, default=32)
    ap.add_argument("--ref-build-workers", type=int, default=4,
                    help="reference arm: heads built concurrently (each ood_build with "
                         "nproc / workers threads)")
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


def ncu_summary(name="ncu_search_summary.json"):
    """A committed ncu summary under profiles/ (dram bytes per launch of a
    line's dominant kernel, from a --set full / dram metrics capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic():
    return (ncu_summary("ncu_search_summary_r2.json") or ncu_summary()).get("dram_bytes_per_launch")


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def timed(fn, stream, flush=None):
    """Device time of fn() on `stream` (CUDA events), L2 flushed before."""
    import torch
    if flush is not None:
        flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)  # no torch.cuda, no code of this package on that path
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2409_10516_b200 as ra
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    flush = torch.empty(a.flush_mb * (1 << 20) // 4, dtype=torch.float32, device=dev)
    parity_jobs = []

    if a.lines_only:
        lines = run_lines(a, ra, flush, stream, dev, parity_jobs,
                          set(a.lines_only.split(",")))
        print(json.dumps({"lines": lines}))
        return

    H, G = a.heads, a.groups
    hpg = H // G
    from paper_2409_10516_b200.shard import OutputGather, groups_for_rank
    by_heads = a.shard == "heads" and world > 1
    my_groups = (groups_for_rank(G, world, rank) if by_heads else list(range(G)))
    layer = rank if not by_heads else 0
    # decode queries: the timed steps and the e2e steps
    n_dec = a.warmup + 2 * a.steps + 2
    # synthetic layer l uses seed 7 + l (SURVEY §8 d; the reference has no layers)
    spec = WorkloadSpec(n_ctx=a.n_ctx, d_model=256, d_head=128, n_heads=H, n_kv_groups=G,
                        seed=7 + layer, n_decode=n_dec)
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
        if rank == 0:
            keys_host.append(w["keys"].cpu().numpy())
            vals_host.append(w["values"].cpu().numpy())
        del w
    setup_s = time.time() - t0
    Hl = len(graphs)
    Q = torch.stack(dq, dim=1).contiguous()  # [n_dec, Hl, d]: Q[i] is one step, contiguous
    del dq
    cfg = ra.EngineConfig(128, 512, a.top_k, a.ef)

    eng = ra.Engine(kvs, graphs, cfg)
    gather = OutputGather(G, hpg, 128, world, rank, dev) if (dist is not None and by_heads) else None
    gather_ms = []

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
    times, search_ms, scanned, expanded = [], [], [], []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(a.warmup, a.warmup + a.steps):
            times.append(timed(lambda: step(i), stream, flush))
            search_ms.append(eng.last_timing()[0])
            s, e = eng.last_stats()
            scanned.append(s)
            expanded.append(e)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
        if gather is not None:  # NCCL all_gather latency alone (per step)
            out0 = eng.decode_step_device(Q[a.warmup])[0]
            torch.cuda.synchronize()
            for _ in range(5):
                gather_ms.append(timed(lambda: gather(out0, dist), stream))

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

        def host_step():
            eng.ctx.bind_stream()
            ra.api._check(ra.lib.ra_engine_step_host(eng.h, qh.data_ptr(), out_h.data_ptr(),
                                                     om_h.data_ptr(), sc_h.data_ptr()))
        e2e.append(timed(host_step, stream))

    out32 = eng.decode_step_device(Q[a.warmup])[0].cpu().numpy()
    bf16 = (bf16_mode(a, ra, spec, my_groups, hpg, Q, cfg, flush, stream, out32, graphs)
            if not a.no_bf16 else None)

    ms = statistics.mean(times)
    ms_search = statistics.mean(search_ms)
    ms_e2e = statistics.mean(e2e)
    shard_balance = None
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
        if gather_ms:
            shard_balance["nccl_all_gather_ms"] = round(statistics.mean(gather_ms), 4)
    d, M = 128, a.max_degree
    bytes_search = statistics.mean([s * d * 4 + e * M * 4 + 0.0 for s, e in zip(scanned, expanded)])
    fused = eng.kernels_per_step() == 1
    if fused:  # the kernel also computes the attention: W's K and V rows (algorithmically
        # once per KV group; the kernel reads them per head) and the Omega V rows
        nW = min(128, a.n_ctx) + min(512, max(a.n_ctx - 128, 0))
        bytes_search += len(my_groups) * nW * d * 8 + Hl * a.top_k * d * 4
    peak, peak_kind = measured_peaks()
    achieved = bytes_search / (ms_search * 1e-3) / 1e9
    layer_tokens = world if (dist is not None and not by_heads) else 1
    res = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms/token", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "strong" if by_heads else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: the reference OOD generator (workload.cpp:102-203) restated on "
                "the GPU, seed 7 + layer",
        "config": workload_config(a, H, G),
        "execution": ("one ra_engine step per token (fused search + attention kernel)"
                      if fused else "one ra_engine step per token (3 kernels)") +
                     (f"; {world} ranks each decode their own layer per step "
                      f"({layer_tokens} layer-tokens per step)" if layer_tokens > 1 else ""),
        "e2e": {"value": round(ms_e2e, 4), "unit": "ms/token",
                "h2d_bytes_per_step": Hl * 128 * 4,
                "d2h_bytes_per_step": Hl * 128 * 8 + Hl * max(eng.k, 1) * 4 + Hl * 8},
        "gpu_launches": eng.kernels_per_step() * a.steps,
        "roofline": {"bound": "hbm",
                     "kernel": "k_graph_search_pipe (latency mode" +
                               (", fused attention: search + W / Omega partials + merge)"
                                if fused else ")"),
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 5), "peak_source": peak_kind,
                     "traffic": ncu_traffic(),
                     "algorithmic_bytes_per_launch": int(bytes_search),
                     "kernel_ms": round(ms_search, 4)},
        "search": {"mean_scanned_per_head": statistics.mean(scanned) / Hl,
                   "mean_expanded_per_head": statistics.mean(expanded) / Hl,
                   "scan_fraction": statistics.mean(scanned) / Hl / (a.n_ctx - 640)},
        "clocks": clk.summary(),
        "shard_balance": shard_balance,
        "bf16_kv": bf16,
        "setup_s": round(setup_s, 1),
        "build_ms_per_head": round(statistics.mean(build_ms), 1),
        "build_phase_ms_per_head": {
            k: round(statistics.mean(g.build_stats.ms[k] for g in graphs), 2)
            for k in ("knn", "knn_tensor", "edges", "prune", "entry", "repair")},
        "build_knn_rows_exact_fallback": sum(g.build_stats.knn_rows_widened for g in graphs),
        # configs[3] (index construction): the layer's graphs built back to back
        # on this GPU (128K prefill queries -> 128K keys per query head)
        "build_layer": {"heads": len(build_ms), "ms_total": round(sum(build_ms), 1),
                        "ms_per_head_median": round(statistics.median(build_ms), 1),
                        "knn_tflops_algorithmic": round(
                            2.0 * a.n_ctx * a.n_ctx * 128 / (statistics.median(
                                [g.build_stats.ms["knn_tensor"] for g in graphs]) * 1e-3) / 1e12, 1)},
    }
    if layer_tokens > 1:
        res["layer_tokens_per_s"] = round(layer_tokens / (ms * 1e-3), 1)
    if rank == 0:
        res["recall"] = recall(eng, graphs, kvs, Q, a, ra)
    del eng
    # the further lines (their own KV and graphs; the headline's memory is kept small)
    if world == 1:
        want = set()
        if not a.no_layers32:
            want.add("layers32")
        if not a.no_batch8:
            want.add("batch8")
        if not a.no_1m:
            want.add("ctx_1m")
        res["lines"] = run_lines(a, ra, flush, stream, dev, parity_jobs, want)
    if rank == 0:
        if world == 1 and not a.no_cpu_baseline:
            res["cpu_baseline"], res["parity"] = cpu_baseline(a, keys_host, vals_host, graphs,
                                                              Q, cfg, parity_jobs)
            res["dropin"] = dropin_decode(a, res["e2e"]["value"])
        print(json.dumps(res))
    if dist is not None:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# multi-context lines: many independent (context, KV group) sets in HBM
# ---------------------------------------------------------------------------
def run_lines(a, ra, flush, stream, dev, parity_jobs, want):
    out = {}
    L = a.line_layers
    if "layers32" in want:
        # north-star shape: layer l = synthetic seed 7 + l, all 8 KV groups
        ctxs = [(l, 7 + l, g) for l in range(L) for g in range(a.groups)]
        out["layers32"] = multi_context_line(
            a, ra, "layers32", ctxs, a.groups, a.n_ctx, flush, stream, dev, parity_jobs,
            f"north-star shape: {L} distinct synthetic layers (seed 7 + l) x {a.groups} KV "
            f"groups x {a.heads // a.groups} Q heads, {a.n_ctx} ctx, batch 1; one token = "
            f"{L * a.heads} searches + sparse attention")
    if "batch8" in want:
        # configs[2] at 8 GPUs, heads sharded: this GPU owns KV group 0 of every
        # layer for all 8 batch items; item b of layer l = seed 7 + 100 b + l
        ctxs = [(l, 7 + 100 * b + l, 0) for l in range(L) for b in range(8)]
        out["batch8"] = multi_context_line(
            a, ra, "batch8", ctxs, 8, a.n_ctx, flush, stream, dev, parity_jobs,
            f"configs[2] per-GPU shard at 8 GPUs: {L} layers x KV group 0 x 8 distinct batch "
            f"contexts (seed 7 + 100 b + l) x {a.heads // a.groups} Q heads, {a.n_ctx} ctx; "
            f"one decode step = {L * 8 * (a.heads // a.groups)} searches + attention")
    if "ctx_1m" in want:
        ctxs = [(0, 7, g) for g in range(a.groups)]
        out["ctx_1m"] = multi_context_line(
            a, ra, "ctx_1m", ctxs, a.groups, 1 << 20, flush, stream, dev, parity_jobs,
            f"configs[4] on one GPU: one full layer ({a.groups} KV groups x "
            f"{a.heads // a.groups} Q heads) at a 1,048,576-token context, batch 1",
            samples=(0, a.groups - 1))
    return out


def multi_context_line(a, ra, name, ctxs, per_layer, n_ctx, flush, stream, dev, parity_jobs,
                       desc, samples=None):
    """Build every (layer, seed, group) context's KV group and its 4 query-head
    graphs on the GPU, then time (i) the layer-batched step - one engine step
    over all heads - and (ii) the layer-serial step - one engine step per
    layer, back to back (the decode dependency chain). Sampled contexts are
    queued for the reference parity check (cpu_baseline leg)."""
    import torch
    from paper_2409_10516_b200.workload import WorkloadSpec, generate_group
    hpg = a.heads // a.groups
    n_dec = a.warmup + a.steps + 1
    bp = ra.OODGraphBuildParams(a.k_train, a.max_degree, a.ef_construction, 8)
    cfg = ra.EngineConfig(128, 512, a.top_k, a.ef)
    if samples is None:  # 8 contexts spread over the line (32 heads)
        samples = tuple(sorted({int(round(i * (len(ctxs) - 1) / 7)) for i in range(8)}))
    t0 = time.time()
    kvs, graphs, qs, host = [], [], [], {}
    build_ms = []
    for ci, (l, seed, g) in enumerate(ctxs):
        spec = WorkloadSpec(n_ctx=n_ctx, d_model=256, d_head=128, n_heads=a.heads,
                            n_kv_groups=a.groups, seed=seed, n_decode=n_dec)
        w = generate_group(spec, g, dev)
        kv = ra.KVGroup(w["keys"], w["values"])
        kvs.append(kv)
        for m in range(hpg):
            tb = time.time()
            graphs.append(ra.ood_build(kv, w["prefill_q"][m], bp))
            build_ms.append((time.time() - tb) * 1e3)
            qs.append(w["decode_q"][m])
        if ci in samples:
            host[ci] = (w["keys"].cpu().numpy(), w["values"].cpu().numpy())
        del w
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    Q = torch.stack(qs, dim=1).contiguous()  # [n_dec, heads, d]
    del qs
    n_l = len(ctxs) // per_layer
    hl = per_layer * hpg  # heads per layer
    eng = ra.Engine(kvs, graphs, cfg)
    per = [ra.Engine(kvs[i * per_layer:(i + 1) * per_layer], graphs[i * hl:(i + 1) * hl], cfg)
           for i in range(n_l)] if n_l > 1 else [eng]

    def serial(i):
        for j, e in enumerate(per):
            e.decode_step_device(Q[i, j * hl:(j + 1) * hl])

    for i in range(a.warmup):
        eng.decode_step_device(Q[i])
        serial(i)
    eng.last_timing(), eng.last_stats()
    torch.cuda.synchronize()
    t_b, s_b, sc, ex, t_s = [], [], [], [], []
    with ClockSampler(dev.index or 0) as clk:
        for i in range(a.warmup, a.warmup + a.steps):
            t_b.append(timed(lambda: eng.decode_step_device(Q[i]), stream, flush))
            s_b.append(eng.last_timing()[0])
            s_, e_ = eng.last_stats()
            sc.append(s_)
            ex.append(e_)
        for i in range(a.warmup, a.warmup + a.steps):
            t_s.append(timed(lambda: serial(i), stream, flush))
    i0 = a.warmup
    out, om, scn = (x.cpu().numpy() for x in eng.decode_step_device(Q[i0]))
    for ci in sorted(host):
        hs = slice(ci * hpg, (ci + 1) * hpg)
        parity_jobs.append({"line": name, "ctx": ci, "keys": host[ci][0], "values": host[ci][1],
                            "blobs": [g.serialize() for g in graphs[hs]],
                            "q": Q[i0, hs].cpu().numpy(), "out": out[hs],
                            "omega": om[hs].view(np.uint32), "scanned": scn[hs],
                            "cfg": cfg})
    nH = len(graphs)
    d, M = 128, a.max_degree
    k = eng.k
    by_search = statistics.mean([s_ * d * 4 + e_ * M * 4 for s_, e_ in zip(sc, ex)])
    nW = min(128, n_ctx) + min(512, max(n_ctx - 128, 0))
    by_attn = len(ctxs) * nW * d * 8 + nH * k * d * 4  # W K+V once per group, Omega V rows
    fused = eng.kernels_per_step() == 1
    by_kernel = by_search + (by_attn if fused else 0)  # the fused kernel also does attention
    ms_b, ms_s, ms_ser = statistics.mean(t_b), statistics.mean(s_b), statistics.mean(t_s)
    peak, kind = measured_peaks()
    gbs = by_kernel / (ms_s * 1e-3) / 1e9
    summ = ncu_summary(f"ncu_{name}_summary.json")
    traffic = summ.get("dram_bytes_per_launch")
    res = {
        "workload": desc, "contexts": len(ctxs), "heads": nH, "n_ctx": n_ctx,
        "value": round(ms_b, 4), "unit": "ms/step (layer-batched: one engine step over all "
                                           "heads)",
        "step_ms_all": [round(x, 4) for x in t_b], "kernel_ms_all": [round(x, 4) for x in s_b],
        "layer_serial_ms": round(ms_ser, 4),
        "layer_serial_note": f"{n_l} engine steps of {hl} heads back to back (the layer "
                             "dependency chain of real decode)",
        "tokens_per_step": 8 if name == "batch8" else 1,
        "searches_per_s": round(nH / (ms_b * 1e-3), 1),
        "kernels_per_step_batched": eng.kernels_per_step(),
        "roofline": {"bound": "hbm", "kernel": "k_graph_search_pipe (" +
                     ("latency mode, fused attention" if fused else "search only") + ")",
                     "achieved": round(gbs, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(gbs / peak, 4), "peak_source": kind, "traffic": traffic,
                     "traffic_over_algorithmic": (round(traffic / by_kernel, 3)
                                                  if traffic else None),
                     "algorithmic_bytes_per_launch": int(by_kernel),
                     "kernel_ms": round(ms_s, 4)},
        "step_GBps": round((by_search + by_attn) / (ms_b * 1e-3) / 1e9, 1),
        "step_frac": round((by_search + by_attn) / (ms_b * 1e-3) / 1e9 / peak, 4),
        "attention_bytes_per_step": int(by_attn),
        "mean_scanned_per_head": round(statistics.mean(sc) / nH, 1),
        "mean_expanded_per_head": round(statistics.mean(ex) / nH, 1),
        "clocks": clk.summary(), "setup_s": round(setup_s, 1),
        "build_ms_per_head": round(statistics.mean(build_ms), 2),
        "hbm_resident_bytes": int(len(ctxs) * n_ctx * d * 8 +
                                  sum(g.device_bytes() for g in graphs)),
    }
    if summ:
        res["roofline"]["ncu"] = {k2: v for k2, v in summ.items() if k2 != "dram_bytes_per_launch"}
    del per, eng, kvs, graphs, Q
    import gc
    gc.collect()
    torch.cuda.synchronize()
    return res


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
        del eng
        res[mode] = {"value": round(statistics.mean(times), 4), "unit": "ms/token",
                     "search_ms": round(statistics.mean(s_ms), 4),
                     "search_GBps": round(by / (statistics.mean(s_ms) * 1e-3) / 1e9, 1),
                     "out_rel_vs_f32": {"max": float(rel.max()), "mean": float(rel.mean())}}
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


def _ref_engine(keys_host, vals_host, blobs, cfg, threads):
    from oracle.ffi import Oracle, available
    if not available("ref"):
        return None, None
    o = Oracle("ref")
    eng = o.engine(np.stack(keys_host), np.stack(vals_host), blobs, cfg.s_init, cfg.s_local,
                   cfg.top_k, -1 if cfg.search_param is None else cfg.search_param, threads)
    return o, eng


def cpu_baseline(a, keys_host, vals_host, graphs, Q, cfg, parity_jobs):
    """CPU baseline leg (rank 0, N=1): the reference's own decode_step
    (oracle/_ref, unmodified sources) on the host cores over the same graphs
    (loaded through OODGraph(keys, blob)), bounded to ~cpu_seconds; plus the
    single-thread latency of one reference OODGraph::search. Doubles as the
    full-size parity check: the headline engine's outputs and every sampled
    head of the further lines against the reference decode_step."""
    import paper_2409_10516_b200 as ra
    threads = os.cpu_count() or 1
    o, reng = _ref_engine(keys_host, vals_host, [g.serialize() for g in graphs], cfg, threads)
    if reng is None:
        return {"value": None, "unavailable": "oracle/_ref not built"}, None
    eng = ra.Engine([g.keys for g in graphs[::cfg_hpg(a)]], graphs, cfg)
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
    del eng
    # single-thread latency of one search (index_oodgraph.cpp:357-411), head 0
    W = ra.static_partition(a.n_ctx, 128, 512).static_set
    og = o.graph(keys_host[0], graphs[0].serialize(), a.ef)
    st = []
    for j in range(min(Q.shape[0], 32)):
        t0 = time.perf_counter()
        og.search(Qh[j, 0], a.top_k, W, a.ef)
        st.append((time.perf_counter() - t0) * 1e3)
    og.close()
    base = {"value": round(statistics.mean(times), 3), "unit": "ms/token", "cores": threads,
            "kind": "reference", "cpu_model": cpu_model(),
            "single_thread_search_ms": round(statistics.median(st), 4),
            "sample": f"{len(times)} decode steps x {Qh.shape[1]} heads at n_ctx {a.n_ctx} "
                      f"(reference decode_step, n_threads={threads}, GPU-built graphs via OODG); "
                      f"single-thread search: median of {len(st)} OODGraph::search calls "
                      f"(k {a.top_k}, ef {a.ef}, Mask W)"}
    parity = None if a.no_parity else {
        "heads_checked": n, "omega_identical": same_om, "scanned_identical": same_sc,
        "max_out_rel_err": max_rel}
    if parity is not None and parity_jobs:
        parity["lines"] = line_parity(o, parity_jobs, threads)
    return base, parity


def dropin_decode(a, e2e_ms):
    """The reference's own API end to end on the GPU backend: the reference
    library with src/index_oodgraph.cpp, attention.cpp and engine.cpp
    replaced by the drop-in TUs (paper_2409_10516_b200/host/*_gpu.cpp over
    libra_b200.so; oracle/_ref/libattnindex_dropin.so): generate_workload
    (seed 7) -> engine_init (ood_build per head, on the GPU) -> decode_step
    per token, timed on the host clock (a synchronous C++ call: host q in,
    TraceEntry out, copies included)."""
    from oracle.ffi import BuildParams, Oracle, available
    if not available("dropin"):
        return {"unavailable": "oracle/_ref/libattnindex_dropin.so not built"}
    o = Oracle("dropin")
    n_dec = a.warmup + a.steps
    t0 = time.time()
    eng, dq, _, _, ms_gen, ms_build = o.engine_from_workload(
        a.n_ctx, a.heads, a.groups, 7, n_dec,
        BuildParams(a.k_train, a.max_degree, a.ef_construction, 8), 128, 512, a.top_k, a.ef,
        os.cpu_count() or 1, 1)
    for i in range(a.warmup):
        eng.step(np.ascontiguousarray(dq[:, i, :]), i)
    times = []
    for i in range(a.warmup, n_dec):
        q = np.ascontiguousarray(dq[:, i, :])
        t1 = time.perf_counter()
        eng.step(q, i)
        times.append((time.perf_counter() - t1) * 1e3)
    ms = statistics.mean(times)
    del eng
    return {"value": round(ms, 4), "unit": "ms/token",
            "vs_ra_engine_step_host": round(ms / e2e_ms, 3) if e2e_ms else None,
            "steps": len(times), "setup_s": round(time.time() - t0, 1),
            "setup_ms": {"generate_workload": round(ms_gen, 1),
                         "engine_init_gpu_builds": round(ms_build, 1)},
            "path": "reference decode_step (engine.cpp:105-115) -> drop-in "
                    "attnindex_engine_gpu.cpp -> ra_engine_step_host (one batched device "
                    "step for all 32 heads), host clock per call"}


def cfg_hpg(a):
    return a.heads // a.groups


def line_parity(o, jobs, threads):
    """Sampled heads of the multi-context lines vs the reference decode_step
    on the same K/V, graphs (OODG blobs) and queries."""
    res = {}
    for j in jobs:
        cfg = j["cfg"]
        reng = o.engine(j["keys"][None], j["values"][None], j["blobs"], cfg.s_init, cfg.s_local,
                        cfg.top_k, -1 if cfg.search_param is None else cfg.search_param, threads)
        rout, rom, rsc = reng.step(np.ascontiguousarray(j["q"]), 0)
        del reng
        r = res.setdefault(j["line"], {"heads_checked": 0, "omega_identical": 0,
                                       "scanned_identical": 0, "max_out_rel_err": 0.0,
                                       "contexts": []})
        om = j["omega"]
        r["heads_checked"] += len(om)
        r["omega_identical"] += int((om == rom[:, : om.shape[1]]).all(axis=1).sum())
        r["scanned_identical"] += int((j["scanned"].astype(np.uint64) == rsc).sum())
        rel = np.linalg.norm(j["out"] - rout, axis=1) / np.linalg.norm(rout, axis=1)
        r["max_out_rel_err"] = max(r["max_out_rel_err"], float(rel.max()))
        r["contexts"].append(j["ctx"])
    return res


def run_reference(a):
    """--impl reference: the reference's own CPU path end to end, rank 0 only.
    oracle/_ref is the unmodified reference sources (Eigen/doctest shims):
    generate_workload (seed 7) -> engine_init's per-head ood_build ->
    decode_step with all host threads. No code of this repo's package, no
    GPU, on this path."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the reference CPU arm runs on rank 0 only
    sys.path.insert(0, ROOT)
    from oracle.ffi import BuildParams, Oracle, available
    if not available("ref"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    threads = os.cpu_count() or 1
    o = Oracle("ref")
    n_dec = a.warmup + a.steps
    t0 = time.time()
    reng, dq, _, _, ms_gen, ms_build = o.engine_from_workload(
        a.n_ctx, a.heads, a.groups, 7, n_dec,
        BuildParams(a.k_train, a.max_degree, a.ef_construction, 8), 128, 512, a.top_k, a.ef,
        threads, a.ref_build_workers)
    setup_s = time.time() - t0
    for i in range(a.warmup):
        reng.step(np.ascontiguousarray(dq[:, i, :]), i)
    times = []
    t_start = time.perf_counter()
    for i in range(a.warmup, a.warmup + a.steps):
        q = np.ascontiguousarray(dq[:, i, :])
        t1 = time.perf_counter()
        reng.step(q, i)
        times.append((time.perf_counter() - t1) * 1e3)
    ms = statistics.mean(times)
    H, G = a.heads, a.groups
    sample = (f"{a.steps} reference decode_steps x {H} heads at n_ctx {a.n_ctx} "
              f"(n_threads={threads}; graphs built by the reference's ood_build)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(ms, 3), "unit": "ms/token",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "strong" if a.shard == "heads" and a.gpus > 1
        else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's own generate_workload (workload.cpp:102-203), "
                "seed 7",
        "config": workload_config(a, H, G),
        "execution": "reference generate_workload + ood_build per head "
                     f"({a.ref_build_workers} heads at a time, {max(1, threads // max(1, a.ref_build_workers))} "
                     "threads each) + decode_step (engine.cpp:105-115) on the host cores "
                     "(oracle/_ref: unmodified reference sources, shimmed Eigen/doctest)",
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/token", "cores": threads,
                         "kind": "reference", "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(ms, 3), "unit": "ms/token", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_start, 2), "setup_s": round(setup_s, 1),
        "setup_ms": {"generate_workload": round(ms_gen, 1), "graph_builds": round(ms_build, 1)}}))


if __name__ == "__main__":
    main()
