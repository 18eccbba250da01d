"""Variant x layout sweep on B200 (the reference's tuner).

    python -m paper_1504_01023_b200.tune --case C3 [--elements N] [--repeats 5] [--out runs.csv]
    python -m paper_1504_01023_b200.tune --case C4 --launch [--out runs.csv]   (tile x CTAs/SM sweep)

Mirror of ``pkg/src/feklab/bench.py:150-196`` (``tune``) and of its CSV schema
(``bench.py:36-52``, so the reference's ``report/`` charts read the output
unchanged).  The reference sweeps storage layout x lane width x worker count
on the CPU.  Here the sweep is layout x lane width x loop-order variant x
geometry path on the GPU; the ``workers`` column holds the GPU count.

This is the extended study (every loop-order variant and geometry path on
device-generated benchmark meshes); ``python -m paper_1504_01023_b200 tune``
is the reference CLI's single-descriptor layout/worker sweep.  ``--launch``
sweeps the two GPU launch knobs the reference's CPU tuner has no analogue for,
for the natural QSS kernel: tile T in {64, 128, 256} elements (template
instantiations, ``fek_batch_desc.tile_elements``) x resident CTAs per SM
(``ctas_per_sm``, 1 .. the occupancy maximum), as two extra CSV columns
(``tile_elements``, ``ctas_per_sm``) after the reference's.

Inputs are generated in HBM by the device mesh generator (``mesh.device_config``)
and re-laid-out on the device.  Each point is the median of ``repeats``
CUDA-event-timed launches, each queued behind an untimed one so the events
bracket the kernel rather than the host-side call overhead.  The model bound is the reference's
``time_bound`` (``perfmodel.py:93-102``) with a B200 profile built from the
MEASURED copy bandwidth and FP64 FMA peak.
"""

from __future__ import annotations

import argparse
import csv
import io
import statistics
import sys

from .bench import CSV_COLUMNS


def b200_profile():
    """(name, bench_bandwidth_gbs, bench_dp_tflops) from the measured peaks."""
    from .measure import flop_peak, hbm_peak

    return "B200 (measured)", hbm_peak()[0], flop_peak(8)[0]


def _interleave(flat, n: int, ds: int, w: int):
    """Element-major flat CUDA tensor -> lane-interleaved (W), NaN-padded tail, on the device."""
    import torch

    blocks = -(-n // w)
    padded = torch.full((blocks * w, ds), float("nan"), dtype=flat.dtype, device=flat.device)
    padded[:n] = flat.view(n, ds)
    return padded.view(blocks, w, ds).transpose(1, 2).contiguous().view(-1)


def sweep(case: str, n_elements: int | None = None, repeats: int = 5, widths=(1, 4, 8, 16, 32, 64),
          variants=("qss", "sqs", "ssq")):
    import torch

    from .kernels.batched import DeviceBatch
    from .kernels.counts import OP_TOTALS, global_accesses
    from .layout import ELEMENT_MAJOR, BatchLayout, LayoutKind
    from .mesh import bench_configs, device_config
    from .problems import GeometryPath, KernelDescriptor, Variant
    from .refelem import ElementType
    from . import integrate_batch

    cfg = bench_configs()[case]
    et, pb = cfg.spec.element_type, cfg.problem
    n = min(n_elements or cfg.spec.n_elements, cfg.spec.n_elements)
    geo, cof = device_config(cfg, 0, n)
    paths = (GeometryPath.GEO_LINEAR, GeometryPath.GEO_GENERIC) if et is ElementType.TETRAHEDRON else \
        (GeometryPath.GEO_GENERIC,)
    _, bw, tf = b200_profile()
    rows = []
    for w in widths:
        if w == 1:
            layout, g, c = ELEMENT_MAJOR, geo, cof
        else:
            layout = BatchLayout(LayoutKind.LANE_INTERLEAVED, w)
            g = _interleave(geo, n, et.geometry_size, w)
            c = _interleave(cof, n, pb.coefficient_size(et), w)
        batch = DeviceBatch(et, pb, n, layout, g, c)
        for v in variants:
            for path in paths:
                desc = KernelDescriptor(Variant(v), path, pb, et)
                A = torch.empty((n, et.n_shape, et.n_shape), dtype=torch.float64, device="cuda")
                b = torch.empty((n, et.n_shape), dtype=torch.float64, device="cuda")
                res = integrate_batch(desc, batch, out=(A, b))  # warm-up + error check
                times = []
                for _ in range(repeats):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    integrate_batch(desc, batch, check=False, out=(A, b))  # keeps the stream busy
                    s.record()
                    integrate_batch(desc, batch, check=False, out=(A, b))
                    e.record()
                    e.synchronize()
                    times.append(s.elapsed_time(e) * 1e6 / n)  # ns per element
                med = statistics.median(times)
                mad = statistics.median(abs(t - med) for t in times)
                acc = global_accesses(et, pb)
                ops = OP_TOTALS[(desc.variant, et, pb)]
                bound = max(acc * 8 / bw, ops / (tf * 1e3))
                rows.append({
                    "variant": v, "geo": path.value, "element": et.value, "problem": pb.value,
                    "layout": layout.kind.value, "lane_width": w, "workers": 1, "n_elements": n,
                    "ns_per_element": f"{med:.4f}", "ns_mad": f"{mad:.4f}",
                    "accesses_per_element": f"{res.traffic.per_element(n):.0f}", "ops_model": ops,
                    "intensity": round(ops / acc), "bound_ns": f"{bound:.4f}",
                    "efficiency_pct": round(bound / med * 100),
                })
        del batch
    return rows


LAUNCH_COLUMNS = list(CSV_COLUMNS) + ["tile_elements", "ctas_per_sm"]


def sweep_launch(case: str, n_elements: int | None = None, repeats: int = 5, tiles=(64, 128, 256)):
    """Tile size x CTAs/SM for the case's natural QSS descriptor, element-major inputs in HBM."""
    import torch

    from . import integrate_batch, launch_config
    from .kernels.batched import DeviceBatch
    from .kernels.counts import OP_TOTALS, global_accesses
    from .layout import ELEMENT_MAJOR
    from .mesh import bench_configs, device_config
    from .problems import KernelDescriptor, Variant, natural_path

    cfg = bench_configs()[case]
    et, pb = cfg.spec.element_type, cfg.problem
    n = min(n_elements or cfg.spec.n_elements, cfg.spec.n_elements)
    geo, cof = device_config(cfg, 0, n)
    batch = DeviceBatch(et, pb, n, ELEMENT_MAJOR, geo, cof)
    desc = KernelDescriptor(Variant.QSS, natural_path(et), pb, et)
    _, bw, tf = b200_profile()
    acc = global_accesses(et, pb)
    ops = OP_TOTALS[(desc.variant, et, pb)]
    bound = max(acc * 8 / bw, ops / (tf * 1e3))
    A = torch.empty((n, et.n_shape, et.n_shape), dtype=torch.float64, device="cuda")
    b = torch.empty((n, et.n_shape), dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    rows = []
    for tile in tiles:
        full = launch_config(desc, ELEMENT_MAJOR, n, tile=tile)
        max_ctas = max(1, min(full["grid"] // sms, 8))
        for ctas in range(1, max_ctas + 1):
            res = integrate_batch(desc, batch, out=(A, b), tile=tile, ctas_per_sm=ctas)
            times = []
            for _ in range(repeats):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                integrate_batch(desc, batch, check=False, out=(A, b), tile=tile, ctas_per_sm=ctas)
                s.record()
                integrate_batch(desc, batch, check=False, out=(A, b), tile=tile, ctas_per_sm=ctas)
                e.record()
                e.synchronize()
                times.append(s.elapsed_time(e) * 1e6 / n)
            med = statistics.median(times)
            mad = statistics.median(abs(t - med) for t in times)
            rows.append({
                "variant": "qss", "geo": desc.geometry_path.value, "element": et.value, "problem": pb.value,
                "layout": "element_major", "lane_width": 1, "workers": 1, "n_elements": n,
                "ns_per_element": f"{med:.4f}", "ns_mad": f"{mad:.4f}",
                "accesses_per_element": f"{res.traffic.per_element(n):.0f}", "ops_model": ops,
                "intensity": round(ops / acc), "bound_ns": f"{bound:.4f}",
                "efficiency_pct": round(bound / med * 100), "tile_elements": tile, "ctas_per_sm": ctas,
            })
    return rows


def best(rows):
    """First-tie-wins minimum of ns_per_element (bench.py:187)."""
    return min(rows, key=lambda r: float(r["ns_per_element"]))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--case", default="C3")
    ap.add_argument("--elements", type=int, default=None)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--launch", action="store_true", help="tile x CTAs/SM sweep of the natural QSS kernel")
    args = ap.parse_args(argv)
    if args.launch:
        rows = sweep_launch(args.case, args.elements, args.repeats)
    else:
        rows = sweep(args.case, args.elements, args.repeats)
    buf = io.StringIO()
    wr = csv.DictWriter(buf, fieldnames=LAUNCH_COLUMNS if args.launch else CSV_COLUMNS)
    wr.writeheader()
    wr.writerows(rows)
    text = buf.getvalue()
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
    sys.stdout.write(text)
    b = best(rows)
    knobs = f" T={b['tile_elements']} CTAs/SM={b['ctas_per_sm']}" if args.launch else ""
    print(f"# best: {b['variant']}/{b['geo']} {b['layout']} W={b['lane_width']}{knobs} {b['ns_per_element']} ns/elem "
          f"({b['efficiency_pct']}% of the B200 bound)", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
