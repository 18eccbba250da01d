#!/usr/bin/env python
"""Pageable vs page-locked host batches through integrate_batch (C5 shard, N=1): copy-thread sweep.

    python tools/e2e_pageable.py [--threads 4,8,12,16]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", default="4,8,12,16")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--chunks", default="0")
    ap.add_argument("--streams", default="3")
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_1504_01023_b200 import ElementBatch, integrate_batch
    from paper_1504_01023_b200.kernels import batched as KB
    from paper_1504_01023_b200.layout import ELEMENT_MAJOR

    parts = [bench.Part(*c) for c in bench.c5_parts(1, 0)]
    pinned, plain = [], []
    for p in parts:
        g = p.geo.view(p.n, -1).cpu().numpy()
        c = p.cof.view(p.n, -1).cpu().numpy()
        pinned.append(ElementBatch.from_arrays(p.desc.element, p.desc.problem, g, c))
        plain.append(ElementBatch(p.desc.element, p.desc.problem, p.n, ELEMENT_MAJOR, g.reshape(-1), c.reshape(-1)))
    del parts

    def step(batches):
        res = [None, None]
        t0 = time.perf_counter()
        for i, b in enumerate(batches):
            res[i] = integrate_batch(bench.Part.__init__ and KB.coerce_descriptor(
                bench.c5_parts(1, 0)[i][1]), b)
        return time.perf_counter() - t0

    step(pinned)
    print(f"pinned: {min(step(pinned) for _ in range(args.reps)) * 1e3:.1f} ms", flush=True)
    from concurrent.futures import ThreadPoolExecutor

    descs = [KB.coerce_descriptor(c[1]) for c in bench.c5_parts(1, 0)]

    def step_concurrent(batches):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(len(batches)) as ex:
            list(ex.map(lambda ib: integrate_batch(descs[ib[0]], ib[1]), enumerate(batches)))
        return time.perf_counter() - t0

    step_concurrent(pinned)
    print(f"pinned, both batches concurrently (two host threads): "
          f"{min(step_concurrent(pinned) for _ in range(args.reps)) * 1e3:.1f} ms", flush=True)
    step_concurrent(plain)
    print(f"pageable, both batches concurrently: {min(step_concurrent(plain) for _ in range(args.reps)) * 1e3:.1f} ms",
          flush=True)
    orig = KB.host_chunk_elements
    orig_streams = KB.HOST_STREAMS
    for ch in [int(x) for x in args.chunks.split(",")]:
        KB.host_chunk_elements = (lambda n, ch=ch: ch) if ch else orig
        for ns in [int(x) for x in args.streams.split(",")]:
            KB.HOST_STREAMS = ns
            KB._stream_cache.clear()
            step(pinned)
            print(f"pinned chunk={ch or 'default'} streams={ns}: {min(step(pinned) for _ in range(args.reps)) * 1e3:.1f} ms",
                  flush=True)
        KB.HOST_STREAMS = orig_streams
        KB._stream_cache.clear()
        for t in [int(x) for x in args.threads.split(",")]:
            KB._copy_threads = lambda t=t: t
            step(plain)
            print(f"pageable chunk={ch or 'default'} threads={t}: {min(step(plain) for _ in range(args.reps)) * 1e3:.1f} ms",
                  flush=True)


if __name__ == "__main__":
    main()
