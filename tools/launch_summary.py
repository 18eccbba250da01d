#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into a markdown table.

    python tools/launch_summary.py gpurun_out/launches_r01.csv "command line" > profiles/launches_r01_summary.md
"""
import collections
import csv
import sys


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    k_i, v_i, u_i = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[k_i]].append(float(r[v_i].replace(",", "")) * scale.get(r[u_i], 1.0))
    total = sum(sum(v) for v in agg.values()) or 1.0
    print(f"Launch list of `{cmd}` under `ncu --metrics gpu__time_duration.sum --clock-control none`")
    print("(cold-cache and serialised: compare shares, not absolute times).\n")
    print("| launches | mean us | share of GPU time | kernel |")
    print("|---|---|---|---|")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f}% | `{name[:90]}` |")


if __name__ == "__main__":
    main()
