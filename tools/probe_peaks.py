#!/usr/bin/env python
"""Measure the B200 numbers the roofline needs but MEASURED_PEAKS.json lacks.

* FP64 FMA peak (independent DFMA chains on all SMs), with the SM clock seen;
* pinned PCIe H2D / D2H / bidirectional copy bandwidth (the e2e ceiling).

Writes gpurun_out/peaks.json; the committed copy is profiles/peaks_r01.json.
"""
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    import pynvml
    import torch

    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libfekprobe.so"))
    out = {}
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    clocks = []
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.01)

    ms, tf = ctypes.c_float(), ctypes.c_double()
    best = 0.0
    for blocks in (sms * 4, sms * 8):
        clocks.clear()
        stop.clear()
        th = threading.Thread(target=sample)
        th.start()
        vals = []
        for _ in range(3):
            assert lib.probe_fp64_peak(blocks, 200000, ctypes.byref(ms), ctypes.byref(tf)) == 0
            vals.append(tf.value)
        stop.set()
        th.join()
        best = max(best, max(vals))
        out[f"fp64_blocks_{blocks}"] = {"tflops": vals, "ms_last": ms.value,
                                        "sm_mhz_median": sorted(clocks)[len(clocks) // 2] if clocks else None}
    out["fp64_tflops_best"] = best
    vals = []
    for _ in range(3):
        assert lib.probe_fp32_peak(sms * 8, 200000, ctypes.byref(ms), ctypes.byref(tf)) == 0
        vals.append(tf.value)
    out["fp32_tflops"] = vals
    out["fp32_tflops_best"] = max(vals)
    out["sms"] = sms

    n = 1 << 30
    hbuf = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    hbuf2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(n, dtype=torch.uint8, device="cuda")
    dbuf2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t

    dbuf.copy_(hbuf, non_blocking=True)
    t_h2d = min(timed(lambda: dbuf.copy_(hbuf, non_blocking=True)) for _ in range(3))
    t_d2h = min(timed(lambda: hbuf2.copy_(dbuf2, non_blocking=True)) for _ in range(3))

    def both():
        with torch.cuda.stream(s1):
            dbuf.copy_(hbuf, non_blocking=True)
        with torch.cuda.stream(s2):
            hbuf2.copy_(dbuf2, non_blocking=True)

    t_bi = min(timed(both) for _ in range(3))
    out["pcie_h2d_gbs"] = n / t_h2d / 1e9
    out["pcie_d2h_gbs"] = n / t_d2h / 1e9
    out["pcie_bidir_gbs_total"] = 2 * n / t_bi / 1e9
    try:
        out["nvidia_smi_pcie"] = subprocess.run(
            ["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max",
             "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except Exception:
        pass
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "peaks.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    sys.exit(main())
