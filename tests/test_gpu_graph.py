"""integrate_batch inside a CUDA graph (device batches, check=False).

The launch-bound use -- the same batch shape integrated again and again with
new data in the same buffers -- is captured once and replayed: every replay
must give the eager result for the data currently in the input buffers, and
the kernel's tile queue (allocated inside the capture, zeroed by the captured
fill) must work on every replay.
"""

import numpy as np
import pytest

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
