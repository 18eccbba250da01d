#!/usr/bin/env python
"""Summarise ncu reports into profiles/ncu_summary.json (+ a markdown table).

    python tools/ncu_summary.py TAG=gpurun_out/prof_C2.ncu-rep ... [--md profiles/ncu_r01.md]

Run here (no GPU): reads the .ncu-rep files with `ncu -i --page raw --csv`.
The JSON is keyed by capture (benchmark configuration, e.g. C5P, C4f32); each record names its
kernel tag (descriptor_dtype) and element count, from which bench.py scales roofline.traffic
(DRAM bytes per element x the launch's elements).
"""
import argparse
import csv
import io
import json
import os
import subprocess

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", None),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", None),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", None),
    "local_loads": ("smsp__sass_inst_executed_op_local_ld.sum", None),
    "inst_executed": ("smsp__inst_executed.sum", None),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", None),
}
UNITS = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    rec = {"kernel": vals[hdr.index("Kernel Name")]}
    for key, (metric, _) in METRICS.items():
        if metric not in hdr:
            continue
        i = hdr.index(metric)
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if key.endswith("_bytes") and u in UNITS:
            v *= UNITS[u]
        if key == "duration_us" and u in UNITS:
            v *= UNITS[u]
        rec[key] = v
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(vals[i])
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    rec["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    rec["dram_bytes_per_launch"] = rec.get("dram_read_bytes", 0) + rec.get("dram_write_bytes", 0)
    rec.update(executed_flops(rep))
    return rec


def executed_flops(rep):
    """Executed FP64/FP32 flops per launch from the SASS source page (FMA counted as 2, FFMA2 as 4)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next((r for r in rows if "Source" in r and "Thread Instructions Executed" in r), None)
    if hdr is None:
        return {}
    isrc, ithr = hdr.index("Source"), hdr.index("Thread Instructions Executed")
    weights = {"DFMA": ("fp64", 2), "DMUL": ("fp64", 1), "DADD": ("fp64", 1),
               "FFMA2": ("fp32", 4), "FMUL2": ("fp32", 2), "FADD2": ("fp32", 2),
               "FFMA": ("fp32", 2), "FMUL": ("fp32", 1), "FADD": ("fp32", 1)}
    tot = {"fp64": 0.0, "fp32": 0.0}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= max(isrc, ithr):
            continue
        words = r[isrc].split()
        if not words:
            continue
        op = (words[1] if words[0].startswith("@") and len(words) > 1 else words[0]).split(".")[0]
        if op in weights:
            kind, w = weights[op]
            try:
                tot[kind] += w * float(r[ithr].replace(",", ""))
            except ValueError:
                pass
    return {"executed_fp64_flops": tot["fp64"], "executed_fp32_flops": tot["fp32"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+", help="TAG=path.ncu-rep")
    ap.add_argument("--out", default="profiles/ncu_summary.json")
    ap.add_argument("--md", default=None)
    args = ap.parse_args()
    data = {}
    if os.path.exists(args.out):
        data = json.load(open(args.out))
    import re
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1504_01023_b200 import mesh

    for item in args.reports:
        tag, rep = item.split("=", 1)
        rec = read(rep)
        rec["report"] = os.path.basename(rep)
        # configuration of the capture (tools/profile_case.py --case KEY [--dtype f32]) and its kernel tag
        cfg_key = re.sub(r"f32$", "", tag)
        cfg = mesh.bench_configs().get(cfg_key)
        if cfg is not None:
            et, pb = cfg.spec.element_type.value, cfg.problem.value
            path = "linear" if et == "tet" else "generic"
            rec["elements"] = cfg.spec.n_elements
            rec["kernel_tag"] = f"qss_{path}_{et}_{pb}_{'f32' if tag.endswith('f32') else 'f64'}"
        data[tag] = rec
    with open(args.out, "w") as fh:
        json.dump(data, fh, indent=1)
    if args.md:
        lines = ["| capture | us | DRAM R+W (MB) | DRAM % peak | FP64 pipe % | FMA pipe % | executed TFLOP/s "
                 "(FMA = 2) | warps active % | regs | top stalls |",
                 "|---|---|---|---|---|---|---|---|---|---|"]
        for tag, r in data.items():
            st = ", ".join(f"{k} {v}%" for k, v in list(r["stall_pct"].items())[:4])
            lines.append(f"| {tag} | {r.get('duration_us', 0):.1f} | {r['dram_bytes_per_launch'] / 1e6:.1f} | "
                         f"{r.get('dram_pct_peak', 0):.1f} | {r.get('fp64_pipe_pct', 0):.1f} | "
                         f"{r.get('fma_pipe_pct', 0):.1f} | "
                         f"{(r.get('executed_fp64_flops', 0) + r.get('executed_fp32_flops', 0)) / (r.get('duration_us', 1) * 1e6):.1f} | "
                         f"{r.get('warps_active_pct', 0):.1f} | {r.get('registers', 0):.0f} | {st} |")
        open(args.md, "w").write("\n".join(lines) + "\n")
    print(json.dumps(data, indent=1)[:3000])


if __name__ == "__main__":
    main()
