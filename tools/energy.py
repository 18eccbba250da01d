#!/usr/bin/env python
"""Energy per element of the C5 kernels under sustained load (NVML energy counter).

    python tools/energy.py [--seconds 3]

For the idle GPU, the tet shard (C5T), the prism shard (C5P) and the whole C5 step: back-to-back
launches for `seconds` after a 1 s warm-up, with NVML's total-energy counter read around the
window.  Prints mean board power, median SM clock, throttle reasons, launches per second and
nJ per element.  Under the board's power cap the step's throughput is set by its energy per
element, not by the kernels' latency hiding.
"""
import argparse
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    args = ap.parse_args()
    import numpy as np
    import pynvml
    import torch

    import bench

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    parts = [bench.Part(*c) for c in bench.c5_parts(1, 0)]
    names = {"SW_POWER_CAP": pynvml.nvmlClocksEventReasonSwPowerCap,
             "HW_SLOWDOWN": pynvml.nvmlClocksEventReasonHwSlowdown,
             "SW_THERMAL": pynvml.nvmlClocksEventReasonSwThermalSlowdown}

    def run(label, fns, n_elems):
        clocks, reasons, stop = [], set(), threading.Event()

        def sample():
            while not stop.is_set():
                clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                reasons.update(k for k, v in names.items() if r & v)
                time.sleep(0.01)

        t_end = time.time() + 1.0
        while fns and time.time() < t_end:  # warm-up into the steady (capped) state
            for f in fns:
                f()
            torch.cuda.synchronize()
        th = threading.Thread(target=sample)
        th.start()
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        t0 = time.time()
        k = 0
        while time.time() - t0 < args.seconds:
            if fns:
                for _ in range(10):
                    for f in fns:
                        f()
                k += 10
                torch.cuda.synchronize()
            else:
                time.sleep(0.05)
        dt = time.time() - t0
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        stop.set()
        th.join()
        joules = (e1 - e0) / 1e3
        line = f"{label:5s}: {joules / dt:6.1f} W, SM {np.median(clocks):.0f} MHz {sorted(reasons)}"
        if fns:
            line += (f", {k / dt:7.1f} launches/s = {k * n_elems / dt / 1e9:5.2f} G elements/s, "
                     f"{joules / (k * n_elems) * 1e9:5.1f} nJ/element")
        print(line, flush=True)
        return joules / dt

    idle = run("idle", [], 0)
    # HBM energy per byte: a device-to-device copy of 2 GiB (read + write bytes)
    src = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    moved = 2 * src.numel() * 8
    w_copy = run("copy", [lambda: dst.copy_(src)], moved)  # "elements" = bytes moved
    del src, dst
    torch.cuda.empty_cache()
    for p in parts:
        run(p.cfg.key, [p.L], p.n)
    run("C5", [p.L for p in parts], sum(p.n for p in parts))
    print(f"(idle board power {idle:.0f} W included in every figure; for `copy` the 'elements' are bytes moved, "
          f"so nJ/element there is nJ per byte)")


if __name__ == "__main__":
    main()
