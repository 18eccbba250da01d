#!/usr/bin/env python
"""Per-launch times of 40-60 back-to-back launches with NVML power/clock samples (DESIGN 5.5).

    python tools/sustained_clocks.py C4 C2 C3
"""
import os, sys, time, threading
sys.path.insert(0, os.getcwd())
import numpy as np, torch, pynvml
from bench import Launcher
from paper_1504_01023_b200 import KernelDescriptor, mesh, natural_path
from paper_1504_01023_b200.problems import Variant
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
print("power limit W", pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000, "default", pynvml.nvmlDeviceGetPowerManagementDefaultLimit(h) / 1000)
samples = []
stop = threading.Event()
def samp():
    while not stop.is_set():
        try:
            samples.append((time.perf_counter(), pynvml.nvmlDeviceGetPowerUsage(h) / 1000,
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                            pynvml.nvmlDeviceGetTemperature(h, 0)))
        except Exception as e:
            samples.append((time.perf_counter(), str(e)))
        time.sleep(0.001)
for case in sys.argv[1:]:
    cfg = mesh.bench_configs()[case]
    et, pb = cfg.spec.element_type, cfg.problem
    desc = KernelDescriptor(Variant.QSS, natural_path(et), pb, et)
    geo, cof = mesh.device_config(cfg)
    L = Launcher(desc, geo, cof)
    L(); torch.cuda.synchronize(); time.sleep(0.5)
    samples.clear(); stop.clear()
    th = threading.Thread(target=samp); th.start()
    t0 = time.perf_counter()
    n = max(40, int(0.2 / 0.00025)) if case != "C4" else 60
    es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for s, e in es:
        s.record(); L(); e.record()
    torch.cuda.synchronize()
    stop.set(); th.join()
    t = [s.elapsed_time(e) for s, e in es]
    q = len(t) // 6
    print(case, "launch ms by sixth:", " ".join(f"{np.mean(t[i*q:(i+1)*q]):.4f}" for i in range(6)))
    ok = [x for x in samples if len(x) == 6]
    for i in range(0, len(ok), max(1, len(ok) // 12)):
        ts, p, sm, mem, r, tmp = ok[i]
        print(f"  t={1e3*(ts-t0):7.1f} ms  P={p:6.1f} W  sm={sm} mem={mem} reasons={r:#x} T={tmp}C")
    del L, geo, cof; torch.cuda.empty_cache(); time.sleep(1.0)
