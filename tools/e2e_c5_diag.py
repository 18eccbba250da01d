#!/usr/bin/env python
"""Where the C5 e2e step goes: each integrate_batch call against the raw PCIe copies of its bytes.

    python tools/e2e_c5_diag.py [--reps 3]

Per part (tets, prisms; N=1 shards, page-locked host batches): the integrate_batch call, the H2D of
its inputs alone, the D2H of its outputs alone and both at once (two streams, 256 MiB pieces, the
same page-locked memory).  Then the whole step serial (bench.py's e2e) and with the two calls on two
host threads, against the step's own bidirectional copy floor.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from concurrent.futures import ThreadPoolExecutor

    import torch

    import bench
    from paper_1504_01023_b200 import ElementBatch, hostmem, integrate_batch

    parts = [bench.Part(*c) for c in bench.c5_parts(1, 0)]
    descs = [p.desc for p in parts]
    batches, outs = [], []
    for p in parts:
        g = p.geo.view(p.n, -1).cpu().numpy()
        c = p.cof.view(p.n, -1).cpu().numpy()
        batches.append(ElementBatch.from_arrays(p.desc.element, p.desc.problem, g, c))
        ns = p.desc.element.n_shape
        outs.append(hostmem.empty(p.n * (ns * ns + ns)))
    del parts
    torch.cuda.empty_cache()
    piece = 256 << 20
    dev = torch.empty(max(max(b.geometry_data.nbytes + b.coefficient_data.nbytes for b in batches),
                          max(o.nbytes for o in outs)) // 8 + 1, dtype=torch.float64, device="cuda")
    dev2 = torch.empty_like(dev)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def copies(srcs, dst, h2d):
        # srcs: host arrays (H2D) or one host array (D2H) moved in 256 MiB pieces on one stream
        st = s_in if h2d else s_out
        with torch.cuda.stream(st):
            off = 0
            for a in srcs:
                t = torch.from_numpy(a.reshape(-1)).view(torch.uint8)
                d = (dev if h2d else dev2).view(torch.uint8)
                for lo in range(0, t.numel(), piece):
                    hi = min(t.numel(), lo + piece)
                    if h2d:
                        d[lo:hi].copy_(t[lo:hi], non_blocking=True)
                    else:
                        t[lo:hi].copy_(d[lo:hi], non_blocking=True)
                off += t.numel()

    def timed(fn):
        best = 1e9
        for _ in range(args.reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best * 1e3

    tot_in = tot_out = 0
    for d, b, o in zip(descs, batches, outs):
        inb = b.geometry_data.nbytes + b.coefficient_data.nbytes
        tot_in += inb
        tot_out += o.nbytes
        h = timed(lambda: copies([b.geometry_data, b.coefficient_data], None, True))
        dd = timed(lambda: copies([o], None, False))
        both = timed(lambda: (copies([b.geometry_data, b.coefficient_data], None, True), copies([o], None, False)))
        call = timed(lambda: integrate_batch(d, b))
        print(f"{d.element.value}: in {inb / 1e9:.2f} GB, out {o.nbytes / 1e9:.2f} GB | H2D {h:.1f} ms "
              f"({inb / h / 1e6:.1f} GB/s), D2H {dd:.1f} ms ({o.nbytes / dd / 1e6:.1f} GB/s), both {both:.1f} ms | "
              f"integrate_batch {call:.1f} ms = {both / call:.2f} of its floor", flush=True)

    def floor():
        copies([x for b in batches for x in (b.geometry_data, b.coefficient_data)], None, True)
        copies(outs, None, False)

    fl = timed(floor)

    def serial():
        for d, b in zip(descs, batches):
            integrate_batch(d, b)

    def concurrent():
        with ThreadPoolExecutor(2) as ex:
            list(ex.map(lambda i: integrate_batch(descs[i], batches[i]), range(2)))

    se, co = timed(serial), timed(concurrent)
    print(f"step: in {tot_in / 1e9:.2f} GB, out {tot_out / 1e9:.2f} GB, bidirectional floor {fl:.1f} ms | serial "
          f"{se:.1f} ms ({fl / se:.2f}), two host threads {co:.1f} ms ({fl / co:.2f})", flush=True)


if __name__ == "__main__":
    main()
