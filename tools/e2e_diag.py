#!/usr/bin/env python
"""Break down the end-to-end (host buffers) integrate_batch time on the C2 workload."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_1504_01023_b200 import ElementBatch, KernelDescriptor, _native, hostmem, integrate_batch, mesh
    from paper_1504_01023_b200.kernels import batched as B
    from paper_1504_01023_b200.problems import GeometryPath, Variant

    cfg = mesh.bench_configs()["C2"]
    geo, cof = mesh.config_rows(cfg)
    et, pb = cfg.spec.element_type, cfg.problem
    hb = ElementBatch.from_arrays(et, pb, geo, cof)
    desc = KernelDescriptor(Variant.QSS, GeometryPath.GEO_LINEAR, pb, et)
    print("input pinned:", hostmem.is_pinned(hb.geometry_data), hostmem.is_pinned(hb.coefficient_data))
    t = time.perf_counter()
    A = hostmem.empty((hb.n_elements, 4, 4))
    print("alloc pinned A ms", (time.perf_counter() - t) * 1e3, "pinned:", hostmem.is_pinned(A))

    def wall(fn, k=3):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts) * 1e3

    # raw torch copies of the same pinned host arrays
    g_t = torch.from_numpy(hb.geometry_data)
    c_t = torch.from_numpy(hb.coefficient_data)
    dg = torch.empty_like(g_t, device="cuda")
    dc = torch.empty_like(c_t, device="cuda")
    print("torch H2D geo+coef ms", wall(lambda: (dg.copy_(g_t, non_blocking=True), dc.copy_(c_t, non_blocking=True))))
    print("integrate_batch e2e ms (min of 3)", wall(lambda: integrate_batch(desc, hb)))
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        integrate_batch(desc, hb)
        ts.append((time.perf_counter() - t0) * 1e3)
    print("integrate_batch e2e ms over 10 calls: mean %.2f min %.2f max %.2f" % (np.mean(ts), np.min(ts), np.max(ts)))
    # the PCIe bound of the step: the same byte counts in both directions at once
    n = hb.n_elements
    out_h = hostmem.empty((n, 20))
    out_d = torch.empty((n, 20), dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o_t = torch.from_numpy(out_h)

    def both():
        with torch.cuda.stream(s1):
            dg.copy_(g_t, non_blocking=True)
            dc.copy_(c_t, non_blocking=True)
        with torch.cuda.stream(s2):
            o_t.copy_(out_d, non_blocking=True)
        s1.synchronize()
        s2.synchronize()
    print("torch H2D inputs || D2H outputs ms", wall(both))

    lib = _native.load()
    n = hb.n_elements
    Ah = hostmem.empty((n, 4, 4))
    bh = hostmem.empty((n, 4))
    dd = B._desc_struct(desc, hb.layout, n, 0, 0, hb.geometry_data.ctypes.data, hb.coefficient_data.ctypes.data,
                        Ah.ctypes.data, bh.ctypes.data, 0)
    for nstreams in (2, 3, 4):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        handles = (ctypes.c_void_p * nstreams)(*[s.cuda_stream for s in streams])
        for chunk in (1 << 18, 1 << 19, 1 << 20):
            ws = lib.fek_host_workspace_bytes(ctypes.byref(dd), nstreams, chunk)
            wsb = torch.empty(ws, dtype=torch.uint8, device="cuda")
            key = ctypes.c_ulonglong()

            def run():
                rc = lib.fek_integrate_host(ctypes.byref(dd), wsb.data_ptr(), ws, nstreams, handles, chunk,
                                            ctypes.byref(key))
                assert rc == 0, rc

            ms = wall(run)
            gbs = (hb.geometry_data.nbytes + hb.coefficient_data.nbytes + Ah.nbytes + bh.nbytes) / ms / 1e6
            print(f"fek_integrate_host streams={nstreams} chunk={chunk:7d}: {ms:7.2f} ms  {gbs:6.1f} GB/s total")
    print("max |A - A_e2e|:", float(np.abs(Ah - integrate_batch(desc, hb).stiffness).max()))


if __name__ == "__main__":
    main()
