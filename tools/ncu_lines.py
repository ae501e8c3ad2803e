#!/usr/bin/env python3
"""Aggregate an ncu source-page CSV (SASS view) by CUDA source line using the
line table of `nvdisasm -g` output for the same kernel (profiling aid).

  python tools/ncu_lines.py <src.csv> <kernel.sass> <divisor> [top]
"""
import collections
import csv
import re
import sys


def main():
    src_csv, sass, div = sys.argv[1], sys.argv[2], float(sys.argv[3])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(src_csv)))
    hdr, data = rows[1], rows[2:]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex, iss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    stall = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    base = int(data[0][ia], 16)
    a2l, cur = {}, None
    for line in open(sass):
        m = re.search(r'File "([^"]+)", line (\d+)', line)
        if m and line.strip().startswith("//"):
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*)", line)
        if m:
            a2l[int(m.group(1), 16)] = cur
    files = {}
    per, samp, reasons = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    tot_s = collections.Counter()
    for r in data:
        key = a2l.get(int(r[ia], 16) - base)
        per[key] += float(r[iex] or 0) / div
        samp[key] += float(r[iss] or 0)
        for h, i in stall.items():
            v = float(r[i] or 0)
            reasons[key][h] += v
            tot_s[h] += v
    print(f"instructions per unit: {sum(per.values()):.1f}   samples: {sum(samp.values()):.0f}")
    print("stalls:", ", ".join(f"{h[6:]}={v:.0f}" for h, v in tot_s.most_common(8)))
    for key, c in per.most_common(top):
        f, ln = key if key else ("?", 0)
        if f not in files:
            try:
                files[f] = open(__import__("glob").glob(f"/root/repo/**/{f}", recursive=True)[0]).read().split("\n")
            except Exception:
                files[f] = []
        txt = files[f][ln - 1].strip()[:70] if files[f] and ln else ""
        rs = ",".join(f"{h[6:]}:{v:.0f}" for h, v in reasons[key].most_common(2) if v)
        print(f"{c:8.1f} samp={samp[key]:5.0f} [{rs}] {f}:{ln} {txt}")


if __name__ == "__main__":
    main()
