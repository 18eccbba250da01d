#!/usr/bin/env python
"""Warp-stall samples of an ncu capture by region of the SASS stream (source page, --import-source).

    python tools/stall_regions.py profiles/prof_C4_r02.ncu-rep [instructions per region]

Prints the capture's stall totals, then consecutive regions of N SASS instructions with their FP64
instruction count and stall samples by reason (wait, math pipe throttle, barrier, long / short
scoreboard, selected, not selected); regions with < 0.4% of the samples are skipped.
"""
import csv
import io
import re
import subprocess
import sys

KEYS = ("samples", "wait", "math", "barrier", "long_sb", "short_sb", "selected", "not_selected")


def main():
    rep = sys.argv[1]
    width = int(sys.argv[2]) if len(sys.argv) > 2 else 80
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if "Source" in r and "stall_wait" in r)
    ix = {k: i for i, k in enumerate(hdr)}
    col = {"samples": "Warp Stall Sampling (All Samples)", **{k: "stall_" + k for k in KEYS[1:]}}
    col["math"] = "stall_math"
    ins = []
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) < len(hdr):
            continue
        rec = {k: float(r[ix[c]] or 0) for k, c in col.items()}
        rec["op"] = r[ix["Source"]].strip()
        rec["opc"] = re.sub(r"^@!?U?P\w+\s+", "", rec["op"]).split(" ")[0].split(".")[0]
        ins.append(rec)
    tot = {k: sum(i[k] for i in ins) for k in KEYS}
    print(f"{rep}: {len(ins)} SASS instructions; stall samples " +
          ", ".join(f"{k} {tot[k] / tot['samples'] * 100:.1f}%" for k in KEYS[1:]))
    print(f"{'first':>5} {'fp64':>4} {'share':>6} " + " ".join(f"{k:>8}" for k in KEYS[1:]) + " | first instruction")
    for s in range(0, len(ins), width):
        seg = ins[s:s + width]
        smp = sum(i["samples"] for i in seg)
        if smp < 0.004 * tot["samples"]:
            continue
        fp = sum(1 for i in seg if i["opc"] in ("DFMA", "DMUL", "DADD"))
        print(f"{s:5d} {fp:4d} {smp / tot['samples'] * 100:5.1f}% " +
              " ".join(f"{sum(i[k] for i in seg) / tot['samples'] * 100:7.1f}%" for k in KEYS[1:]) +
              f" | {seg[0]['op'][:50]}")


if __name__ == "__main__":
    main()
