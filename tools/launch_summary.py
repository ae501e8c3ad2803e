#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, mean duration, share of the process's kernel time.
  python tools/launch_summary.py gpurun_out/launches.csv profiles/launches_r2_summary.json "<command>"
"""
import csv
import json
import sys


def kernel_key(name):
    name = name.replace("void ", "", 1).replace("(anonymous namespace)::", "")
    depth, out = 0, []
    for ch in name:  # cut at the argument list (outside template brackets)
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            break
        out.append(ch)
    return "".join(out)


def main():
    src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.DictReader(l for l in open(src) if not l.startswith("=="))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = {}
    for r in rows:
        k = kernel_key(r["Kernel Name"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", "")) / 1e3
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = {k: {"launches": v[0], "mean_us": round(v[1] / v[0], 2), "share": round(v[1] / tot, 4)}
           for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    json.dump({"command": cmd,
               "note": "ncu serialises launches and runs them cold-cache; compare shares, not absolutes",
               "kernels": out}, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main()
