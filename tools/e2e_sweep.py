#!/usr/bin/env python
"""e2e (host buffers) chunk x stream sweep on C2 against the plain H2D||D2H copy floor (DESIGN 5.4)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1504_01023_b200 import ElementBatch, KernelDescriptor, integrate_batch, mesh, natural_path
from paper_1504_01023_b200.kernels import batched as B
from paper_1504_01023_b200.problems import Variant
cfg = mesh.bench_configs()["C2"]
geo, cof = mesh.config_rows(cfg)
et, pb = cfg.spec.element_type, cfg.problem
hb = ElementBatch.from_arrays(et, pb, geo, cof)
desc = KernelDescriptor(Variant.QSS, natural_path(et), pb, et)
orig = B.host_chunk_elements
def run(chunk, ns, reps=6):
    B.host_chunk_elements = (lambda n: chunk) if chunk else orig
    B.HOST_STREAMS = ns
    B._stream_cache.clear()
    r = integrate_batch(desc, hb); r = integrate_batch(desc, hb); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        r = integrate_batch(desc, hb)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
# plain-copy floor
g = torch.from_numpy(hb.geometry_data); c = torch.from_numpy(hb.coefficient_data)
dg = torch.empty_like(g, device="cuda"); dc = torch.empty_like(c, device="cuda")
A = torch.empty(hb.n_elements * 20, dtype=torch.float64).pin_memory(); dA = torch.empty_like(A, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        dg.copy_(g, non_blocking=True); dc.copy_(c, non_blocking=True)
    with torch.cuda.stream(s2):
        A.copy_(dA, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e.record(); torch.cuda.synchronize()
    print("floor H2D||D2H ms", s.elapsed_time(e), flush=True)
for rep in range(2):
    for chunk in (0, 262144, 131072, 65536):
        for ns in (3, 4):
            print(f"chunk {chunk or 'default'} streams {ns}: {run(chunk, ns):.2f} ms", flush=True)
