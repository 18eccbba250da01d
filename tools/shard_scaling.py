#!/usr/bin/env python
"""Strong-scaling check on ONE GPU: time each rank's C5 shards for world sizes 1, 2, 4, 8.

    python tools/shard_scaling.py [--steps 20] [--warmup 5]

bench.py --gpus N splits both C5 batches by element range (distributed.shard_bounds) and has no
collective on the hot path, so an N-GPU step is the slowest rank's shard step.  This times the
shards of every rank of each world size on the one GPU available (sequentially, graph-timed like
bench.py) and prints the per-rank step times, the projected N-GPU value (64,156,250 / max rank
time) and the parallel efficiency against N=1 -- the kernels' share of strong scaling.  It is not
an N-GPU measurement (no NVLink, no concurrent ranks, one power envelope).  A short timed region
finishes before the board's power cap lowers the clock, which favours small
shards; --equal-time removes that bias.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--equal-time", action="store_true",
                    help="time steps*N steps at world N, so every timed region lasts as long as N=1's "
                         "(same power-cap exposure, DESIGN.md 5.5)")
    args = ap.parse_args()
    import time

    import torch

    import bench

    base = None
    for world in [int(w) for w in args.worlds.split(",")]:
        per_rank = []
        for rank in range(world):
            parts = [bench.Part(*c) for c in bench.c5_parts(world, rank)]

            def step():
                for p in parts:
                    p.L()

            step.launchers = [p.L for p in parts]
            time.sleep(0.3)  # same starting clock state for every rank's measurement
            steps = args.steps * (world if args.equal_time else 1)
            per_rank.append(bench.time_graph([step], steps, args.warmup) / steps)
            del parts, step
            torch.cuda.empty_cache()
        worst = max(per_rank)
        value = bench.C5_TOTAL / (worst / 1e3)
        base = base or value
        print(f"N={world}: rank step ms {' '.join(f'{t:.3f}' for t in per_rank)} -> projected "
              f"{value / 1e9:.2f} G elements/s, efficiency {value / (base * world):.3f}", flush=True)


if __name__ == "__main__":
    main()
