"""Kernel-packed output: integrate_batch(..., packed=True).

The kernel writes BatchResult.flat_output()'s packed rows [A row-major | b]
directly in the requested output layout (element-major or lane-interleaved,
NaN pad lanes).  Must equal the split-array result bit for bit, on the device
and host paths, for every case and lane width.
"""

import numpy as np
import pytest

from conftest import golden
from paper_1504_01023_b200 import (BatchLayout, DeviceBatch, ElementBatch, ElementType, LayoutKind, ProblemClass,
                                   case_descriptors, integrate_batch, pack_rows)

pytestmark = pytest.mark.gpu

CASES = [(ElementType.TETRAHEDRON, ProblemClass.POISSON), (ElementType.TETRAHEDRON, ProblemClass.CONV_DIFF),
         (ElementType.PRISM, ProblemClass.POISSON), (ElementType.PRISM, ProblemClass.CONV_DIFF)]


@pytest.mark.parametrize("et,pb", CASES, ids=lambda c: getattr(c, "value", c))
@pytest.mark.parametrize("w", [1, 4, 16, 64])
def test_packed_equals_split_bitwise(et, pb, w):
    import torch

    z = golden(f"corpus_{et.value}_{pb.value}.npz")
    batch = ElementBatch.from_arrays(et, pb, z["geometry_rows"], z["coefficient_rows"])
    out_layout = BatchLayout(LayoutKind.LANE_INTERLEAVED, w) if w > 1 else BatchLayout(LayoutKind.ELEMENT_MAJOR)
    desc = case_descriptors(et, pb)[0]
    split = integrate_batch(desc, batch)
    want = pack_rows(split.output_rows(), out_layout)  # NaN pads, reference packing
    for b in (batch, DeviceBatch.from_host(batch)):
        res = integrate_batch(desc, b, out_layout=out_layout, packed=True)
        flat = res.flat.cpu().numpy() if isinstance(res.flat, torch.Tensor) else res.flat
        assert flat.shape == want.shape
        assert np.array_equal(flat, want, equal_nan=True)
        assert np.array_equal(np.asarray(res.flat_output() if not isinstance(res.flat, torch.Tensor)
                                         else res.flat_output().cpu()), want, equal_nan=True)
        em = res.element_matrix(5)
        assert np.array_equal(em.A, split.stiffness[5]) and np.array_equal(em.b, split.load[5])


def test_packed_fp32_and_custom_pad():
    import torch

    et, pb = ElementType.PRISM, ProblemClass.CONV_DIFF
    z = golden(f"corpus_{et.value}_{pb.value}.npz")
    batch = ElementBatch.from_arrays(et, pb, z["geometry_rows"], z["coefficient_rows"])
    d32 = DeviceBatch.from_host(batch, dtype=torch.float32)
    desc = case_descriptors(et, pb)[0]
    split = integrate_batch(desc, d32)
    lay = BatchLayout(LayoutKind.LANE_INTERLEAVED, 8)
    res = integrate_batch(desc, d32, out_layout=lay, packed=True)
    want = pack_rows(split.output_rows().double().cpu().numpy(), lay, 0.0)
    got = res.flat_output(pad_value=0.0).double().cpu().numpy()
    assert np.array_equal(got, want)
