#!/usr/bin/env python
"""Per-instruction shared-memory wavefronts of an ncu report (source page, SASS): where do the
bank conflicts that `l1tex__data_bank_conflicts_pipe_lsu_mem_shared` counts come from?

    python tools/smem_conflicts.py gpurun_out/prof_C5T_r02.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if "Source" in r and "L1 Wavefronts Shared" in r)
    i = {k: hdr.index(k) for k in ("Address", "Source", "Instructions Executed", "L1 Wavefronts Shared",
                                   "L1 Wavefronts Shared Ideal", "L1 Wavefronts Shared Excessive")}
    recs = []
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= max(i.values()):
            continue
        try:
            wf = float(r[i["L1 Wavefronts Shared"]] or 0)
            ideal = float(r[i["L1 Wavefronts Shared Ideal"]] or 0)
            ex = float(r[i["L1 Wavefronts Shared Excessive"]] or 0)
            ins = float(r[i["Instructions Executed"]] or 0)
        except ValueError:
            continue
        if wf:
            recs.append((ex, wf, ideal, ins, r[i["Address"]], r[i["Source"]]))
    tot_wf = sum(x[1] for x in recs)
    tot_ex = sum(x[0] for x in recs)
    print(f"{rep}: shared wavefronts {tot_wf:.3e}, excessive {tot_ex:.3e} ({100 * tot_ex / max(tot_wf, 1):.1f}%)")
    by_op = {}
    for ex, wf, ideal, ins, addr, src in recs:
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        a = by_op.setdefault(op, [0, 0, 0])
        a[0] += wf
        a[1] += ideal
        a[2] += ex
    for op, (wf, ideal, ex) in sorted(by_op.items(), key=lambda kv: -kv[1][0]):
        print(f"  {op:24s} wavefronts {wf:.3e} ideal {ideal:.3e} excessive {ex:.3e}")
    print("top instructions by excessive wavefronts:")
    for ex, wf, ideal, ins, addr, src in sorted(recs, reverse=True)[:top]:
        print(f"  {addr} {src[:60]:60s} exec {ins:.3e} wf {wf:.3e} ideal {ideal:.3e} excess {ex:.3e}")


if __name__ == "__main__":
    main()
