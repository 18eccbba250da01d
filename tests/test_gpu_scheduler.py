"""Dynamic tile queue (fek_batch_desc.scheduler, ABI v3).

With a scheduler buffer the persistent CTAs take tiles from an atomic counter
instead of the static round-robin order.  Results must not depend on which CTA
integrated which tile: bit-identical to the static launch, the same
first-error key, and the queue words back at zero after every launch so the
buffer is reusable on the same stream.
"""

import ctypes

import numpy as np
import pytest

from conftest import golden
from paper_1504_01023_b200 import (ELEMENT_MAJOR, BatchLayout, ElementType, LayoutKind, ProblemClass,
                                   case_descriptors, mesh, _native)
from paper_1504_01023_b200.kernels.batched import _desc_struct

pytestmark = pytest.mark.gpu

CASES = [(ElementType.TETRAHEDRON, ProblemClass.POISSON), (ElementType.TETRAHEDRON, ProblemClass.CONV_DIFF),
         (ElementType.PRISM, ProblemClass.POISSON), (ElementType.PRISM, ProblemClass.CONV_DIFF)]


def _launch(desc, geo, cof, sched=None, packed=None, ctas_per_sm=0):
    import torch

    lib = _native.load()
    et = desc.element
    ns = et.n_shape
    n = geo.numel() // et.geometry_size
    err = torch.full((1,), -1, dtype=torch.int64, device=geo.device)
    if packed is None:
        A = torch.empty((n, ns, ns), dtype=geo.dtype, device=geo.device)
        b = torch.empty((n, ns), dtype=geo.dtype, device=geo.device)
        ptrs = (A.data_ptr(), b.data_ptr())
        out = (A, b)
    else:
        from paper_1504_01023_b200 import flat_length

        flat = torch.empty(flat_length(n, ns * ns + ns, packed), dtype=geo.dtype, device=geo.device)
        ptrs = (flat.data_ptr(), 0)
        out = (flat,)
    dtype = _native.DTYPE["float64" if geo.dtype == torch.float64 else "float32"]
    d = _desc_struct(desc, ELEMENT_MAJOR, n, 0, dtype, geo.data_ptr(), cof.data_ptr(), ptrs[0], ptrs[1],
                     err.data_ptr(), out_layout=packed)
    d.scheduler = sched.data_ptr() if sched is not None else None
    d.ctas_per_sm = ctas_per_sm
    _native.check(lib.fek_integrate(ctypes.byref(d), torch.cuda.current_stream().cuda_stream), "fek_integrate")
    torch.cuda.synchronize()
    return out, int(err.item()) & 0xFFFFFFFFFFFFFFFF


def _equal(x, y):
    import torch

    return all(torch.equal(torch.nan_to_num(a, nan=7.0), torch.nan_to_num(b, nan=7.0)) for a, b in zip(x, y))


@pytest.mark.parametrize("et,pb", CASES, ids=lambda c: getattr(c, "value", c))
def test_dynamic_equals_static_bitwise(et, pb):
    import torch

    z = golden(f"corpus_{et.value}_{pb.value}.npz")
    # corpus tiled up to ~300k elements: many tiles per CTA, ragged last tile
    reps = 300_000 // z["geometry_rows"].shape[0] + 1
    geo = torch.from_numpy(np.tile(z["geometry_rows"], (reps, 1))[:299_977]).cuda()
    cof = torch.from_numpy(np.tile(z["coefficient_rows"], (reps, 1))[:299_977]).cuda()
    sched = torch.zeros(2, dtype=torch.int64, device="cuda")
    for desc in case_descriptors(et, pb):
        ref, key_s = _launch(desc, geo, cof)
        for cap in (0, 1):
            got, key_d = _launch(desc, geo, cof, sched, ctas_per_sm=cap)
            assert _equal(ref, got), (desc.short_name(), cap)
            assert key_d == key_s
            assert sched.tolist() == [0, 0]  # reset by the last CTA -> reusable
        lay = BatchLayout(LayoutKind.LANE_INTERLEAVED, 16)
        ps, _ = _launch(desc, geo, cof, packed=lay)
        pd, _ = _launch(desc, geo, cof, sched, packed=lay)
        assert _equal(ps, pd) and sched.tolist() == [0, 0]


def test_dynamic_first_error_rule():
    """Several bad elements spread over many tiles: the reported one is the static launch's."""
    import torch

    et, pb = ElementType.PRISM, ProblemClass.CONV_DIFF
    cfg = mesh.bench_configs()["C4"]  # prism ConvDiff
    geo, cof = mesh.device_config(cfg, 0, 1 << 20)
    geo = geo.view(-1, et.geometry_size).clone()
    for e in (999_999, 700_001, 4_100_000 % (1 << 20), 655_360):
        geo[e] = geo[e].view(6, 3)[[0, 2, 1, 3, 5, 4]].reshape(-1)  # inverted prism
    desc = case_descriptors(et, pb)[0]
    sched = torch.zeros(2, dtype=torch.int64, device="cuda")
    _, key_s = _launch(desc, geo.view(-1), cof)
    _, key_d = _launch(desc, geo.view(-1), cof, sched)
    assert key_s != 0xFFFFFFFFFFFFFFFF and key_d == key_s
    assert _native.decode_error(key_d)[0] == 655_360 - 0  # first bad block wins, then smallest index
    assert sched.tolist() == [0, 0]


def test_dynamic_on_generated_mesh_repeated():
    """The same queue buffer across back-to-back launches on one stream (C1 size)."""
    import torch

    cfg = mesh.bench_configs()["C1"]
    geo, cof = mesh.device_config(cfg)
    desc = case_descriptors(cfg.spec.element_type, cfg.problem)[0]
    sched = torch.zeros(2, dtype=torch.int64, device="cuda")
    ref, _ = _launch(desc, geo, cof)
    for _ in range(3):
        got, key = _launch(desc, geo, cof, sched)
        assert _equal(ref, got) and key == 0xFFFFFFFFFFFFFFFF


def test_scheduler_alignment_checked():
    import torch

    lib = _native.load()
    et, pb = ElementType.TETRAHEDRON, ProblemClass.POISSON
    desc = case_descriptors(et, pb)[0]
    geo = torch.zeros(128 * 12, dtype=torch.float64, device="cuda")
    cof = torch.zeros(128 * 4, dtype=torch.float64, device="cuda")
    A = torch.empty(128 * 16, dtype=torch.float64, device="cuda")
    b = torch.empty(128 * 4, dtype=torch.float64, device="cuda")
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    sched = torch.zeros(4, dtype=torch.int64, device="cuda")
    d = _desc_struct(desc, ELEMENT_MAJOR, 128, 0, _native.DTYPE["float64"], geo.data_ptr(), cof.data_ptr(),
                     A.data_ptr(), b.data_ptr(), err.data_ptr())
    d.scheduler = sched.data_ptr() + 4
    assert lib.fek_integrate(ctypes.byref(d), None) == _native.ERR_ALIGNMENT
