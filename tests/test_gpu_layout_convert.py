"""On-device layout conversion: DeviceBatch.convert / fek_convert_layout.

Mirrors the reference's layout tests (test_layout.py round trips, convert
content preservation, NaN pad lanes) on arrays already in HBM: every pair of
storage schemes, ragged sizes, fp64 and fp32, compared bit for bit with the
host ``convert`` (the reference's pack_rows/unpack_rows restated), and the
integrals of a converted batch bit-identical to the original's.
"""

import numpy as np
import pytest

from conftest import golden
from paper_1504_01023_b200 import (BatchLayout, DeviceBatch, ElementBatch, ElementType, LayoutKind, ProblemClass,
                                   case_descriptors, convert, integrate_batch)

pytestmark = pytest.mark.gpu

WIDTHS = [1, 4, 8, 16, 32, 64]


def lay(w):
    return BatchLayout(LayoutKind.ELEMENT_MAJOR) if w == 1 else BatchLayout(LayoutKind.LANE_INTERLEAVED, w)


def host_batch(et, pb, n, w):
    z = golden(f"corpus_{et.value}_{pb.value}.npz")
    reps = n // z["geometry_rows"].shape[0] + 1
    geo = np.tile(z["geometry_rows"], (reps, 1))[:n]
    cof = np.tile(z["coefficient_rows"], (reps, 1))[:n]
    return ElementBatch.from_arrays(et, pb, geo, cof, lay(w))


@pytest.mark.parametrize("n", [1, 127, 1000, 4099])
@pytest.mark.parametrize("w_in", WIDTHS)
def test_convert_all_pairs_bitwise(n, w_in):
    import torch

    et, pb = ElementType.PRISM, ProblemClass.CONV_DIFF
    hb = host_batch(et, pb, n, w_in)
    db = DeviceBatch.from_host(hb)
    for w_out in WIDTHS:
        want = convert(hb, lay(w_out))
        got = convert(db, lay(w_out))
        assert isinstance(got, DeviceBatch) and got.layout == lay(w_out)
        for a, b in ((got.geometry_data, want.geometry_data), (got.coefficient_data, want.coefficient_data)):
            assert np.array_equal(a.cpu().numpy(), b, equal_nan=True), (w_in, w_out)
        # fp32 arrays convert the same way (values are exact casts)
        g32 = DeviceBatch.from_host(hb, dtype=torch.float32).convert(lay(w_out), pad_value=-7.0)
        want32 = convert(hb, lay(w_out), pad_value=-7.0)
        assert np.array_equal(g32.geometry_data.cpu().numpy(), want32.geometry_data.astype(np.float32), equal_nan=True)


def test_convert_round_trip_and_copy_semantics():
    hb = host_batch(ElementType.TETRAHEDRON, ProblemClass.POISSON, 999, 8)
    db = DeviceBatch.from_host(hb)
    same = db.convert(lay(8))
    assert same.geometry_data.data_ptr() != db.geometry_data.data_ptr()  # a copy, as the reference returns
    back = db.convert(lay(1)).convert(lay(64)).convert(lay(8))
    assert np.array_equal(back.geometry_data.cpu().numpy(), hb.geometry_data, equal_nan=True)
    assert np.array_equal(back.to_host().coefficient_data, hb.coefficient_data, equal_nan=True)


@pytest.mark.parametrize("et,pb", [(ElementType.TETRAHEDRON, ProblemClass.CONV_DIFF),
                                   (ElementType.PRISM, ProblemClass.POISSON)], ids=lambda c: getattr(c, "value", c))
def test_integrals_independent_of_converted_layout(et, pb):
    import torch

    hb = host_batch(et, pb, 3001, 1)
    db = DeviceBatch.from_host(hb)
    desc = case_descriptors(et, pb)[0]
    ref = integrate_batch(desc, db)
    for w in (4, 32):
        res = integrate_batch(desc, db.convert(lay(w)))
        assert torch.equal(res.stiffness, ref.stiffness) and torch.equal(res.load, ref.load)


def test_convert_argument_errors():
    from paper_1504_01023_b200 import _native

    lib = _native.load()
    assert lib.fek_convert_layout(None, 3, None, 1, 10, 12, 0, 0.0, None) == _native.ERR_ARGUMENT
    assert lib.fek_convert_layout(None, 1, None, 1, 10, 43, 0, 0.0, None) == _native.ERR_ARGUMENT
    assert lib.fek_convert_layout(None, 1, None, 1, 0, 12, 0, 0.0, None) == _native.OK


def test_convert_unaligned_arrays_take_the_plain_kernel():
    """Arrays offset by one fp32 word (not 16-byte aligned) use the plain-load kernel: same bytes."""
    import torch

    hb = host_batch(ElementType.PRISM, ProblemClass.POISSON, 1001, 4)
    db = DeviceBatch.from_host(hb, dtype=torch.float32)

    def shifted(t):
        buf = torch.empty(t.numel() + 1, dtype=t.dtype, device=t.device)
        view = buf[1:]
        view.copy_(t)
        return view

    odd = DeviceBatch(db.element_type, db.problem, db.n_elements, db.layout,
                      shifted(db.geometry_data), shifted(db.coefficient_data))
    assert odd.geometry_data.data_ptr() % 16 != 0
    for w in (1, 16):
        a, b = odd.convert(lay(w)), db.convert(lay(w))
        assert torch.equal(torch.nan_to_num(a.geometry_data, nan=5.0), torch.nan_to_num(b.geometry_data, nan=5.0))
        assert torch.equal(torch.nan_to_num(a.coefficient_data, nan=5.0),
                           torch.nan_to_num(b.coefficient_data, nan=5.0))


@pytest.mark.parametrize("w", [1, 8])
def test_fekb_streams_into_device_batch(tmp_path, w):
    """read_batch(path, device=...) streams a FEKB file through pinned staging into HBM."""
    import torch

    from paper_1504_01023_b200 import read_batch, write_batch
    from paper_1504_01023_b200.kernels.batched import _read_device_batch

    hb = host_batch(ElementType.PRISM, ProblemClass.CONV_DIFF, 20_011, w)
    path = tmp_path / "mesh.fekb"
    write_batch(hb, path)
    for db in (read_batch(path, device="cuda"), _read_device_batch(path, "cuda", chunk_bytes=4096 * 8 + 8)):
        assert isinstance(db, DeviceBatch) and db.layout == hb.layout and db.n_elements == hb.n_elements
        assert np.array_equal(db.geometry_data.cpu().numpy(), hb.geometry_data, equal_nan=True)
        assert np.array_equal(db.coefficient_data.cpu().numpy(), hb.coefficient_data, equal_nan=True)
    d32 = _read_device_batch(path, "cuda", dtype=torch.float32, chunk_bytes=1 << 16)
    assert d32.dtype == torch.float32
    assert np.array_equal(d32.geometry_data.cpu().numpy(), hb.geometry_data.astype(np.float32), equal_nan=True)
    desc = case_descriptors(ElementType.PRISM, ProblemClass.CONV_DIFF)[0]
    r1, r2 = integrate_batch(desc, read_batch(path, device="cuda")), integrate_batch(desc, read_batch(path))
    assert np.array_equal(r1.stiffness.cpu().numpy(), r2.stiffness)
