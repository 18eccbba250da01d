#!/usr/bin/env python
"""Bandwidth of the on-device layout conversion (fek_convert_layout) on the C4 geometry + coefficients."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1504_01023_b200 import BatchLayout, DeviceBatch, LayoutKind, mesh
    from paper_1504_01023_b200.layout import ELEMENT_MAJOR

    cfg = mesh.bench_configs()["C4"]
    geo, cof = mesh.device_config(cfg)
    db = DeviceBatch(cfg.spec.element_type, cfg.problem, cfg.spec.n_elements, ELEMENT_MAJOR, geo, cof)
    nbytes = 2 * (geo.numel() + cof.numel()) * 8
    for w_in, w_out in ((1, 32), (32, 1), (4, 64), (1, 4)):
        src = db if w_in == 1 else db.convert(BatchLayout(LayoutKind.LANE_INTERLEAVED, w_in))
        to = ELEMENT_MAJOR if w_out == 1 else BatchLayout(LayoutKind.LANE_INTERLEAVED, w_out)
        for _ in range(3):
            out = src.convert(to)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 10
        for _ in range(reps):
            out = src.convert(to)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"convert W{w_in}->W{w_out}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s (read+write, incl. allocation)")
        del out


if __name__ == "__main__":
    main()
