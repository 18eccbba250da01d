#!/usr/bin/env python
"""Dynamic SASS instruction mix of an ncu report (source page): warp-level instructions executed
per opcode, per element (pass the element count).

    python tools/sass_dyn_mix.py gpurun_out/prof_C4_r02.ncu-rep 16006482 [threads_per_element]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, n = sys.argv[1], int(sys.argv[2])
    tpe = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if "Source" in r and "Thread Instructions Executed" in r)
    isrc, ithr = hdr.index("Source"), hdr.index("Thread Instructions Executed")
    agg = collections.Counter()
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= max(isrc, ithr) or not r[isrc].strip():
            continue
        w = r[isrc].split()
        op = (w[1] if w[0].startswith("@") and len(w) > 1 else w[0])
        base = op.split(".")[0]
        if base in ("IMAD", "MOV") and ("MOV" in op):
            base = "MOV-like"
        try:
            agg[base] += float(r[ithr].replace(",", ""))
        except ValueError:
            pass
    tot = sum(agg.values())
    print(f"{rep}: {tot / n:.0f} thread-instructions per element ({tot / n / tpe:.0f} per thread)")
    for op, v in agg.most_common(30):
        print(f"  {op:12s} {v / n:8.1f} per element  {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
