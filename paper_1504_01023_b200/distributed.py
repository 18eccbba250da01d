"""Multi-GPU sharding: contiguous element ranges, no traffic on the hot path.

Elements are independent (Algorithm 1's element loop), so a
homogeneous batch splits into contiguous ranges exactly like the reference's
worker split ``np.linspace(0, n, workers+1)`` (``batched.py:573``), rounded to
whole lane blocks (and even counts, for 16-byte fp32 TMA rows).  Each rank
integrates its range with ``base_index = lo`` so error indices stay absolute
and the kernel's block/point/element error ordering is global.

Collectives (NCCL over NVLink; gloo in CPU tests) run only AFTER the timed
region, on a few bytes:

* ``all_reduce(SUM)`` of the per-rank verification sums: the uint64
  bit-pattern sums are exactly additive (wrapping integer sums), so their
  reduced value is bitwise the single-GPU value; the fp64 sums (sum A, sum b,
  sum |A|, sum |b|) match it only to rounding (fp64 addition is not
  associative and the per-rank partition differs from ``fek_checksum``'s
  592-block split), so verification gates on the bit-pattern sums and the
  error key;
* ``all_reduce(MIN)`` of the error key (first bad element over all ranks).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native

SIGN = 1 << 63


def shard_bounds(n: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """Contiguous [lo, hi) of rank ``rank``; boundaries are multiples of ``align``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    cut = lambda g: min(n, (n * g // world) // align * align) if g < world else n  # noqa: E731
    return cut(rank), cut(rank + 1)


def all_shards(n: int, world: int, align: int = 128) -> list[tuple[int, int]]:
    return [shard_bounds(n, world, g, align) for g in range(world)]


# ---------------------------------------------------------------------------
# error keys as order-preserving signed ints (NCCL has no uint64 MIN)
# ---------------------------------------------------------------------------

def key_to_signed(key: int) -> int:
    x = int(key) ^ SIGN
    return x - (1 << 64) if x >= SIGN else x


def signed_to_key(v: int) -> int:
    return (int(v) & 0xFFFFFFFFFFFFFFFF) ^ SIGN


def allreduce_error_key(key: int, group=None) -> int:
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([key_to_signed(key)], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return signed_to_key(int(t.item()))


# ---------------------------------------------------------------------------
# verification sums
# ---------------------------------------------------------------------------

def device_checksum(result, base_index: int = 0):
    """(f64[4], int64[2]) CUDA tensors: fek_checksum over a device BatchResult."""
    import torch

    from .kernels.batched import _desc_struct

    lib = _native.load()
    A, b = result.stiffness, result.load
    dtype_code = _native.DTYPE["float64" if A.dtype == torch.float64 else "float32"]
    from .layout import ELEMENT_MAJOR

    dd = _desc_struct(result.descriptor, ELEMENT_MAJOR, result.n_elements, base_index, dtype_code, 0, 0,
                      A.data_ptr(), b.data_ptr(), 0)
    scratch = torch.empty(lib.fek_checksum_scratch_bytes(), dtype=torch.uint8, device=A.device)
    f = torch.empty(4, dtype=torch.float64, device=A.device)
    u = torch.empty(2, dtype=torch.int64, device=A.device)
    _native.check(lib.fek_checksum(ctypes.byref(dd), scratch.data_ptr(), f.data_ptr(), u.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream), "fek_checksum")
    return f, u


def host_checksum(A: np.ndarray, b: np.ndarray, base_index: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """numpy restatement of fek_checksum's bit-pattern sums (for CPU tests / cross-checks)."""
    out_u = np.zeros(2, dtype=np.uint64)
    for j, arr in enumerate((A, b)):
        flat = np.ascontiguousarray(arr).reshape(-1)
        per = flat.size // max(1, A.shape[0]) if A.shape[0] else 0
        bits = flat.view(np.uint64) if flat.dtype == np.float64 else flat.view(np.uint32).astype(np.uint64)
        idx = np.arange(flat.size, dtype=np.uint64) + np.uint64(base_index * per)
        with np.errstate(over="ignore"):
            out_u[j] = np.sum(bits * (np.uint64(2) * idx + np.uint64(1)), dtype=np.uint64)
    f = np.array([A.sum(), b.sum(), np.abs(A).sum(), np.abs(b).sum()], dtype=np.float64)
    return f, out_u


def allreduce_sums(f, u, group=None):
    """SUM-reduce the verification sums across ranks (in place); returns (f, u)."""
    import torch.distributed as dist

    if dist.get_backend(group) != "nccl" and f.is_cuda:  # gloo (CPU tests, one-GPU multi-rank runs)
        fc, uc = f.cpu(), u.cpu()
        dist.all_reduce(fc, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(uc, op=dist.ReduceOp.SUM, group=group)
        f.copy_(fc)
        u.copy_(uc)
        return f, u
    dist.all_reduce(f, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(u, op=dist.ReduceOp.SUM, group=group)
    return f, u


def env_rank() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))
