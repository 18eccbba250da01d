"""Out-of-bounds detection without compute-sanitizer (closed on this pool).

Every array the kernel touches is carved from the middle of a larger buffer:
outputs are surrounded by canary words that must survive the launch
untouched (no stray writes, including the bulk-store tails), inputs by NaN
poison that would surface in the results if a stray read ever fed the math.
Ragged sizes hit partial tiles, odd fp32 prism rows (sub-16-byte tails) and
interleaved padding.
"""

import numpy as np
import pytest

from conftest import golden
from paper_1504_01023_b200 import (BatchLayout, DeviceBatch, ElementType, LayoutKind, ProblemClass,
                                   case_descriptors, flat_length, integrate_batch, pack_rows)

pytestmark = pytest.mark.gpu

GUARD = 4096  # reals on each side
CANARY = -12345.6875  # exactly representable in fp32 and fp64


def _carve(total, dtype, fill):
    import torch

    buf = torch.full((total + 2 * GUARD,), fill, dtype=dtype, device="cuda")
    return buf, buf[GUARD:GUARD + total]


@pytest.mark.parametrize("dtype_name", ["float64", "float32"])
@pytest.mark.parametrize("n", [1, 3, 127, 129, 1001])
@pytest.mark.parametrize("w", [1, 8, 64])
def test_no_stray_reads_or_writes(dtype_name, n, w):
    import torch

    dtype = getattr(torch, dtype_name)
    layout = BatchLayout(LayoutKind.LANE_INTERLEAVED, w) if w > 1 else BatchLayout(LayoutKind.ELEMENT_MAJOR)
    for et, pb in ((ElementType.TETRAHEDRON, ProblemClass.POISSON), (ElementType.TETRAHEDRON, ProblemClass.CONV_DIFF),
                   (ElementType.PRISM, ProblemClass.POISSON), (ElementType.PRISM, ProblemClass.CONV_DIFF)):
        z = golden(f"corpus_{et.value}_{pb.value}.npz")
        idx = np.arange(n) % z["geometry_rows"].shape[0]
        geo = pack_rows(z["geometry_rows"][idx], layout)
        cof = pack_rows(z["coefficient_rows"][idx], layout)
        gbuf, g = _carve(geo.size, dtype, float("nan"))
        cbuf, c = _carve(cof.size, dtype, float("nan"))
        g.copy_(torch.from_numpy(geo))
        c.copy_(torch.from_numpy(cof))
        ns = et.n_shape
        abuf, A = _carve(n * ns * ns, dtype, CANARY)
        bbuf, b = _carve(n * ns, dtype, CANARY)
        batch = DeviceBatch(et, pb, n, layout, g, c)
        for desc in case_descriptors(et, pb):
            integrate_batch(desc, batch, out=(A.view(n, ns, ns), b.view(n, ns)))
            torch.cuda.synchronize()
            for buf, inner in ((abuf, A), (bbuf, b)):
                head, tail = buf[:GUARD], buf[GUARD + inner.numel():]
                assert bool((head == CANARY).all()) and bool((tail == CANARY).all()), (desc.short_name(), n, w)
            assert bool(torch.isfinite(A).all()) and bool(torch.isfinite(b).all()), (desc.short_name(), n, w)
        assert flat_length(n, et.geometry_size, layout) == geo.size
