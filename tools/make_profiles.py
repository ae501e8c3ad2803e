#!/usr/bin/env python3
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

  python tools/make_profiles.py launches <launches.csv> <out.json> <cmd-string>
  python tools/make_profiles.py full <report.ncu-rep> <out.json> <cmd-string> [algorithmic_bytes]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out, cmd):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = collections.defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            per[name].append(float(r["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in per.values())
    res = {"command": cmd,
           "note": "ncu serialises launches and runs them cold-cache; compare shares, not absolutes",
           "kernels": {k: {"launches": len(v), "mean_us": round(sum(v) / len(v), 2),
                           "share": round(sum(v) / tot, 4)} for k, v in
                       sorted(per.items(), key=lambda kv: -sum(kv[1]))}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def full(rep, out, cmd, alg=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = lambda k: vals[hdr.index(k)] if k in hdr else None
    num = lambda k: float(get(k).replace(",", "")) if get(k) not in (None, "") else None
    dur_ns = num("gpu__time_duration.sum")
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    # units of dram bytes may be in KB/MB depending on ncu scaling
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}
    u_rd = units[hdr.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in hdr else "byte"
    u_wr = units[hdr.index("dram__bytes_write.sum")] if "dram__bytes_write.sum" in hdr else "byte"
    u_t = units[hdr.index("gpu__time_duration.sum")]
    tscale = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}[u_t]
    stalls = {}
    for k in hdr:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            v = num(k)
            if v and v > 0.05:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
    res = {"command": cmd, "kernel": get("Kernel Name"), "grid": get("launch__grid_size"),
           "block": get("launch__block_size"), "registers": get("launch__registers_per_thread"),
           "duration_us": dur_ns * tscale if dur_ns else None,
           "dram_bytes_read": rd * scale.get(u_rd, 1) if rd is not None else None,
           "dram_bytes_write": wr * scale.get(u_wr, 1) if wr is not None else None,
           "warp_instructions": num("smsp__inst_executed.sum"),
           "stall_cycles_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])}
    if res["dram_bytes_read"] is not None:
        res["dram_bytes_per_launch"] = res["dram_bytes_read"] + (res["dram_bytes_write"] or 0)
    if alg:
        res["algorithmic_bytes_per_launch"] = float(alg)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(*sys.argv[2:5])
    else:
        full(*sys.argv[2:])
