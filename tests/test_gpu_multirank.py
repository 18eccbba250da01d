"""Two ranks on ONE B200 (gloo, both on cuda:0): the strong-scaled C5 path's multi-rank logic.

bench.py's headline shards both C5 batches by contiguous element range over the ranks
(distributed.shard_bounds = the reference's worker split, batched.py:573) and verifies after
timing with all_reduce(MIN error key) and all_reduce(SUM bit-pattern checksums).  The kernels of
the two ranks never wait on each other (there is no collective on the hot path), so running both
ranks on one GPU exercises exactly the code an 8-GPU run executes, minus NCCL's transport:
* each rank integrates its shard_bounds range with base_index = range start;
* the reduced bit-pattern sums equal a single launch over the whole batch, bit for bit;
* an element made inverted inside rank 1's prism shard wins the MIN error-key reduction
  (absolute element index, quadrature point 0).
"""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

BAD_LOCAL = 1000  # element of rank 1's prism shard made inverted


def _invert(part, local):
    g = part.geo.view(part.n, -1)
    g[local] = -g[local]


def _rank(rank, world, port, out):
    import torch.distributed as dist

    import bench
    from paper_1504_01023_b200.distributed import shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    parts = [bench.Part(*c) for c in bench.c5_parts(world, rank)]
    for p in parts:
        assert (p.lo, p.lo + p.n) == shard_bounds(p.cfg.spec.n_elements, world, rank)
        if rank == 1 and p.cfg.key == "C5P":
            _invert(p, BAD_LOCAL)
        p.L()
    torch.cuda.synchronize()
    ver = bench.c5_verify([(p.desc, p.lo, p.n, p.cfg.key, p.L) for p in parts])
    if rank == 0:
        out.put({k: v for k, v in ver.items() if k != "collectives"})
        out.put({p.cfg.key: (p.lo, p.n) for p in parts})
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_a_single_launch():
    import bench
    from paper_1504_01023_b200 import _native
    from paper_1504_01023_b200.distributed import shard_bounds

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ver2, shards = q.get(timeout=600), q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert shards["C5T"][0] == 0 and shards["C5P"][0] == 0

    # one rank, the whole batches, the same injected element at its absolute index
    parts = [bench.Part(*c) for c in bench.c5_parts(1, 0)]
    lo1, _ = shard_bounds(parts[1].cfg.spec.n_elements, 2, 1)
    _invert(parts[1], lo1 + BAD_LOCAL)
    for p in parts:
        p.L()
    torch.cuda.synchronize()
    for p in parts:
        key = p.L.error_key()
        r2 = ver2[p.cfg.key]
        assert r2["error_key_all_ranks"] == key, p.cfg.key
        from paper_1504_01023_b200.distributed import device_checksum
        from paper_1504_01023_b200.kernels.batched import BatchResult, _traffic

        f, u = device_checksum(BatchResult(p.desc, p.n, p.L.A, p.L.b, _traffic(p.desc, p.n)))
        assert r2["bitsum_A"] == int(u[0].item()) & 0xFFFFFFFFFFFFFFFF, p.cfg.key
        assert r2["bitsum_b"] == int(u[1].item()) & 0xFFFFFFFFFFFFFFFF, p.cfg.key
    assert ver2["C5T"]["error_key_all_ranks"] == _native.NO_ERROR
    element, point, kind = _native.decode_error(ver2["C5P"]["error_key_all_ranks"])
    assert (element, point, kind) == (lo1 + BAD_LOCAL, 0, _native.KIND_INVERTED)
