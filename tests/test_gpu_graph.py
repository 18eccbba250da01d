"""integrate_batch inside a CUDA graph (device batches, check=False).

The launch-bound use -- the same batch shape integrated again and again with
new data in the same buffers -- is captured once and replayed: every replay
must give the eager result for the data currently in the input buffers, and
the kernel's tile queue (allocated inside the capture, zeroed by the captured
fill) must work on every replay.
"""

import numpy as np
import pytest

import paper_1504_01023_b200 as fek
from conftest import golden
from paper_1504_01023_b200 import (DeviceBatch, ElementBatch, ElementType, ProblemClass, case_descriptors,
                                   integrate_batch)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("et,pb", [(ElementType.PRISM, ProblemClass.CONV_DIFF),
                                   (ElementType.TETRAHEDRON, ProblemClass.POISSON)], ids=lambda c: c.value)
def test_capture_and_replay(et, pb):
    import torch

    z = golden(f"corpus_{et.value}_{pb.value}.npz")
    geo, cof = z["geometry_rows"], z["coefficient_rows"]
    n = geo.shape[0]
    db = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof))
    desc = case_descriptors(et, pb)[0]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up outside the capture, as torch recommends
        integrate_batch(desc, db, check=False)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        res = integrate_batch(desc, db, check=False)
    rng = np.random.default_rng(5)
    for k in range(4):
        # new data in the captured buffers: permuted elements, rescaled coefficients
        perm = rng.permutation(n)
        scale = 1.0 + 0.25 * k
        g_k, c_k = geo[perm], cof[perm] * scale
        db.geometry_data.copy_(torch.from_numpy(g_k.reshape(-1)))
        db.coefficient_data.copy_(torch.from_numpy(c_k.reshape(-1)))
        graph.replay()
        torch.cuda.synchronize()
        want = integrate_batch(desc, DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, g_k, c_k)))
        assert torch.equal(res.stiffness, want.stiffness) and torch.equal(res.load, want.load)
        assert int(res.error_word.item()) == -1
        res.check_errors()  # no error: returns
    # an inverted element in the captured buffers: the replay's error word, resolved and raised
    bad = geo.copy()
    bad[7] = -bad[7]
    db.geometry_data.copy_(torch.from_numpy(bad.reshape(-1)))
    graph.replay()
    with pytest.raises(fek.InvertedElement) as err:
        res.check_errors()
    assert err.value.element_index == 7


def test_bench_graph_timing_does_every_step():
    """bench.time_graph: the timed graph replays all K launches over the whole batch.

    Each launcher's outputs are poisoned before the timed replay; afterwards every
    buffer set must hold the eager result bit for bit (no launch skipped or cut
    short), the tile queues must be back at zero, and the replay must take at
    least K x the single-launch time floor of a real kernel.
    """
    import torch

    import bench
    from paper_1504_01023_b200 import KernelDescriptor, mesh, natural_path
    from paper_1504_01023_b200.problems import Variant

    cfg = mesh.bench_configs()["C1"]
    et, pb = cfg.spec.element_type, cfg.problem
    desc = KernelDescriptor(Variant.QSS, natural_path(et), pb, et)
    geo, cof = mesh.device_config(cfg)
    launchers = [bench.Launcher(desc, geo, cof), bench.Launcher(desc, geo.clone(), cof.clone())]
    launchers[0]()
    torch.cuda.synchronize()
    want_A, want_b = launchers[0].A.clone(), launchers[0].b.clone()

    null_ctx = bench._Null

    class Poison(null_ctx):
        def __enter__(self):  # runs right before the timed replay
            for L in launchers:
                L.A.fill_(float("nan"))
                L.b.fill_(float("nan"))
            torch.cuda.synchronize()
            return self

    steps = 6
    ms = bench.time_graph(launchers, steps, 3, sampler=Poison())
    for L in launchers:
        assert torch.equal(L.A, want_A) and torch.equal(L.b, want_b)
        assert L.error_key() == 0xFFFFFFFFFFFFFFFF
        assert L.sched.tolist() == [0, 0]
    # 303 MB per launch cannot move faster than ~8 TB/s
    assert ms / steps >= 0.030, ms
