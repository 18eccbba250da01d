#!/usr/bin/env python
"""Launch one benchmark configuration's integration kernel a few times (for ncu).

    python tools/profile_case.py --case C2 --launches 4 [--dtype f32] [--variant qss]

Inputs are generated on the host and uploaded once; each launch is one
fek_integrate over the whole configuration.  Prints per-launch CUDA-event
times (not valid under a profiler).
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="C2")
    ap.add_argument("--launches", type=int, default=4)
    ap.add_argument("--dtype", default="f64", choices=("f64", "f32"))
    ap.add_argument("--variant", default="qss")
    ap.add_argument("--layout-width", type=int, default=1)
    args = ap.parse_args()

    import torch

    from bench import Launcher
    from paper_1504_01023_b200 import KernelDescriptor, mesh, natural_path
    from paper_1504_01023_b200.layout import BatchLayout, LayoutKind, pack_rows
    from paper_1504_01023_b200.problems import Variant

    cfg = mesh.bench_configs()[args.case]
    et, pb = cfg.spec.element_type, cfg.problem
    desc = KernelDescriptor(Variant(args.variant), natural_path(et), pb, et)
    geo_rows, cof_rows = mesh.config_rows(cfg)
    layout = None
    if args.layout_width > 1:
        layout = BatchLayout(LayoutKind.LANE_INTERLEAVED, args.layout_width)
        g, c = pack_rows(geo_rows, layout), pack_rows(cof_rows, layout)
    else:
        g, c = geo_rows.reshape(-1), cof_rows.reshape(-1)
    dt = torch.float32 if args.dtype == "f32" else torch.float64
    geo = torch.from_numpy(g).to("cuda", dtype=dt)
    cof = torch.from_numpy(c).to("cuda", dtype=dt)
    launch = Launcher(desc, geo, cof, layout=layout)
    times = []
    for _ in range(args.launches):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        launch()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    assert launch.error_key() == 0xFFFFFFFFFFFFFFFF
    # bit-pattern digest of the outputs: equal digests <=> bit-identical results across builds
    ia = launch.A.contiguous().view(-1).view(torch.int32 if dt == torch.float32 else torch.int64).to(torch.int64)
    ib = launch.b.contiguous().view(-1).view(torch.int32 if dt == torch.float32 else torch.int64).to(torch.int64)
    w = torch.arange(1, ia.numel() + 1, device="cuda", dtype=torch.int64)
    digest = int((ia * w).sum().item()) ^ int((ib * w[: ib.numel()]).sum().item())
    print(f"{args.case} {desc.short_name()} {args.dtype} n={launch.n} ms/launch={['%.4f' % t for t in times]} "
          f"digest={digest & 0xFFFFFFFFFFFFFFFF:016x}")


if __name__ == "__main__":
    main()
