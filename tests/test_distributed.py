"""Multi-rank host logic on CPU (gloo, world_size 2): sharding, sums, error keys.

The hot path has no collective; these cover the plumbing around it: shard
bounds reproduce the reference's contiguous worker split, the bit-pattern
verification sums are exactly additive across shards (so an all-reduce of
per-rank sums equals the single-GPU sum bit for bit), and the error key
MIN-reduction returns the globally first bad element.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1504_01023_b200.distributed import (all_shards, host_checksum, key_to_signed, shard_bounds,
                                               signed_to_key)


def test_shard_bounds_cover_and_align():
    for n in (0, 1, 127, 1000, 1_053_696, 16_006_482):
        for world in (1, 2, 3, 4, 8):
            sh = all_shards(n, world)
            assert sh[0][0] == 0 and sh[-1][1] == n
            for (a, b), (c, _) in zip(sh[:-1], sh[1:]):
                assert b == c and a <= b
                assert b % 128 == 0 or b == n


def test_shard_bounds_follow_linspace_split():
    n, world = 10_000_000, 8
    lin = np.linspace(0, n, world + 1).astype(int)
    for g in range(world):
        lo, hi = shard_bounds(n, world, g, align=1)
        assert (lo, hi) == (lin[g], lin[g + 1])


def test_error_key_order_preserved():
    keys = sorted([0, 3, 1 << 40, (1 << 63) - 1, 1 << 63, (1 << 64) - 2, (1 << 64) - 1])
    signed = [key_to_signed(k) for k in keys]
    assert signed == sorted(signed)
    assert [signed_to_key(s) for s in signed] == keys


def test_bit_sums_are_additive_across_shards(rng):
    A = rng.normal(size=(1000, 6, 6))
    b = rng.normal(size=(1000, 6))
    f_all, u_all = host_checksum(A, b)
    u = np.zeros(2, dtype=np.uint64)
    f = np.zeros(4)
    for lo, hi in all_shards(1000, 3, align=8):
        fs, us = host_checksum(A[lo:hi], b[lo:hi], base_index=lo)
        with np.errstate(over="ignore"):
            u += us
        f += fs
    assert np.array_equal(u, u_all)
    assert np.allclose(f, f_all, rtol=1e-12)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, A, b, bad, out):
    import torch
    import torch.distributed as dist

    from paper_1504_01023_b200.distributed import allreduce_error_key, allreduce_sums

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(A.shape[0], world, rank, align=8)
    f, u = host_checksum(A[lo:hi], b[lo:hi], base_index=lo)
    ft = torch.from_numpy(f.copy())
    ut = torch.from_numpy(u.view(np.int64).copy())
    allreduce_sums(ft, ut)
    # each rank reports its own first bad element as a key (point 0, inverted)
    mine = [e for e in bad if lo <= e < hi]
    key = ((min(mine) >> 13) << 24 | (min(mine) & 8191) << 7 | 2) if mine else (1 << 64) - 1
    out[rank] = (ft.numpy().copy(), ut.numpy().view(np.uint64).copy(), allreduce_error_key(key))
    dist.destroy_process_group()


def test_gloo_world2_reductions(rng):
    world = 2
    A = rng.normal(size=(777, 4, 4))
    b = rng.normal(size=(777, 4))
    bad = [700, 9, 400]
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), A, b, bad, out), nprocs=world, start_method="spawn")
    f_all, u_all = host_checksum(A, b)
    for r in range(world):
        f, u, key = out[r]
        assert np.array_equal(u, u_all)
        assert np.allclose(f, f_all, rtol=1e-12)
        assert key == (9 << 7 | 2)
