#!/usr/bin/env python
"""Where does per-launch time go for short cases?  Events per launch vs queued launches vs one CUDA graph."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench import Launcher, time_launches
from paper_1504_01023_b200 import KernelDescriptor, mesh, natural_path
from paper_1504_01023_b200.problems import Variant

for case in sys.argv[1:] or ["C1", "C2", "C3"]:
    cfg = mesh.bench_configs()[case]
    et, pb = cfg.spec.element_type, cfg.problem
    desc = KernelDescriptor(Variant.QSS, natural_path(et), pb, et)
    geo, cof = mesh.device_config(cfg)
    Ls = [Launcher(desc, geo, cof)] + [Launcher(desc, geo.clone(), cof.clone()) for _ in range(2)]
    steps = 30
    per, tot = time_launches(Ls, steps, 5)
    # queued: a sleep kernel first so the host enqueues everything before the GPU starts
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(50_000_000)
    s.record()
    for k in range(steps):
        Ls[k % 3]()
    e.record(); torch.cuda.synchronize()
    q = s.elapsed_time(e) / steps
    # graph of `steps` launches (separate queue buffers per launcher, so replay is safe)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for L in Ls:
            L.stream = st.cuda_stream
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for k in range(steps):
                Ls[k % 3]()
        g.replay(); st.synchronize()
        torch.cuda._sleep(50_000_000)
        s.record(st); g.replay(); e.record(st)
    torch.cuda.synchronize()
    gr = s.elapsed_time(e) / steps
    print(f"{case}: events/launch mean {np.mean(per)*1e3:.1f} us min {np.min(per)*1e3:.1f}; span/steps {tot/steps*1e3:.1f}; "
          f"queued {q*1e3:.1f}; graph {gr*1e3:.1f}", flush=True)
    del Ls, geo, cof; torch.cuda.empty_cache()
