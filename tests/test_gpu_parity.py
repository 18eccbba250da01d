"""GPU parity: libfek.so (sm_100a) against the reference's own outputs and the oracle.

Tolerance (SPEC / north_star): fp64 relative Frobenius <= 1e-12 per element
for A and b (test_acceptance.py:58-64 norm).  Bitwise where the reference
promises bitwise behaviour: layout / worker (here: chunk, shard, path)
independence and batch-vs-element equality (test_kernels.py:240-291).
"""

import numpy as np
import pytest

import paper_1504_01023_b200 as fek
from conftest import GOLDEN, golden
from oracle import numpy_oracle as O
from paper_1504_01023_b200 import (BatchLayout, CoefficientSet, DeviceBatch, ElementBatch, ElementGeometry,
                                   ElementType, GeometryPath, KernelDescriptor, LayoutKind, ProblemClass,
                                   Variant, case_descriptors, integrate_batch, integrate_element)

pytestmark = pytest.mark.gpu

TET, PRISM = ElementType.TETRAHEDRON, ElementType.PRISM
POISSON, CONVDIFF = ProblemClass.POISSON, ProblemClass.CONV_DIFF
CASES = [(TET, POISSON), (PRISM, POISSON), (TET, CONVDIFF), (PRISM, CONVDIFF)]
TOL = 1e-12


def rel(got, want):
    return O.rel_frobenius(np.asarray(got), np.asarray(want))


def corpus(et, pb):
    z = golden(f"corpus_{et.value}_{pb.value}.npz")
    return z, ElementBatch.from_arrays(et, pb, z["geometry_rows"], z["coefficient_rows"])


@pytest.mark.parametrize("et,pb", CASES, ids=lambda c: getattr(c, "value", c))
def test_every_descriptor_matches_reference(et, pb):
    z, batch = corpus(et, pb)
    for desc in case_descriptors(et, pb):
        res = integrate_batch(desc, batch)
        name = desc.short_name()
        assert rel(res.stiffness, z[f"A_{name}"]).max() <= TOL, name
        assert rel(res.load, z[f"b_{name}"]).max() <= TOL, name
        assert rel(res.stiffness, z["A_algorithm1"]).max() <= TOL, name
        assert res.traffic.per_element(batch.n_elements) == fek.global_accesses(et, pb)


@pytest.mark.parametrize("et,pb", CASES, ids=lambda c: getattr(c, "value", c))
def test_device_path_bitwise_equals_host_path(et, pb):
    import torch

    z, batch = corpus(et, pb)
    dbatch = DeviceBatch.from_host(batch)
    for desc in case_descriptors(et, pb):
        host = integrate_batch(desc, batch)
        dev = integrate_batch(desc, dbatch)
        assert isinstance(dev.stiffness, torch.Tensor) and dev.stiffness.is_cuda
        assert np.array_equal(host.stiffness, dev.stiffness.cpu().numpy())
        assert np.array_equal(host.load, dev.load.cpu().numpy())


@pytest.mark.parametrize("et,pb", CASES, ids=lambda c: getattr(c, "value", c))
def test_layout_bitwise_transparency(et, pb):
    z, batch = corpus(et, pb)
    desc = case_descriptors(et, pb)[0]
    base = integrate_batch(desc, batch)
    for w in (1, 4, 8, 16, 32, 64):
        other = ElementBatch.from_arrays(et, pb, z["geometry_rows"], z["coefficient_rows"],
                                         BatchLayout(LayoutKind.LANE_INTERLEAVED, w))
        res = integrate_batch(desc, other)
        assert np.array_equal(base.stiffness, res.stiffness), w
        assert np.array_equal(base.load, res.load), w
        assert np.isfinite(res.stiffness).all()  # NaN padding never leaks


def test_unit_elements_analytic():
    unit = ElementGeometry(TET, TET.reference_vertices)
    G = np.array([[-1.0, -1.0, -1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    for desc in case_descriptors(TET, POISSON):
        em = integrate_element(desc, unit, CoefficientSet.poisson(np.zeros(4)))
        assert np.abs(em.A - G @ G.T / 6.0).max() < 1e-14
        assert np.all(em.b == 0.0)
        em = integrate_element(desc, unit, CoefficientSet.poisson(np.ones(4)))
        assert np.abs(em.b - 1.0 / 24.0).max() < 1e-14
    c = np.zeros((4, 4))
    c[0, 0] = 1.0
    mass = np.full((4, 4), 1.0 / 120.0) + np.eye(4) / 120.0
    for desc in case_descriptors(TET, CONVDIFF):
        em = integrate_element(desc, unit, CoefficientSet.convdiff(c, np.zeros(4)))
        assert np.abs(em.A - mass).max() < 1e-14
    for et in ElementType:
        geom = ElementGeometry(et, et.reference_vertices)
        for v in Variant:
            desc = KernelDescriptor(v, GeometryPath.GEO_GENERIC, CONVDIFF, et)
            em = integrate_element(desc, geom, CoefficientSet.convdiff(np.zeros((4, 4)), np.zeros(4)))
            assert np.all(em.A == 0.0) and np.all(em.b == 0.0)


def test_unit_elements_match_reference():
    z = golden("unit_elements.npz")
    for et in ElementType:
        geom = ElementGeometry(et, et.reference_vertices)
        for pb in ProblemClass:
            coeff = CoefficientSet.poisson(np.ones(et.n_quad)) if pb is POISSON else \
                CoefficientSet.convdiff(np.eye(4), np.ones(4))
            for desc in case_descriptors(et, pb):
                em = integrate_element(desc, geom, coeff)
                assert rel(em.A[None], z[f"A_{desc.short_name()}"][None]).max() <= 1e-14
                assert rel(em.b[None], z[f"b_{desc.short_name()}"][None]).max() <= 1e-14


def test_batch_of_identical_elements_bitwise_equals_element():
    unit = ElementGeometry(TET, TET.reference_vertices)
    coeff = CoefficientSet.poisson(np.zeros(4))
    for desc in case_descriptors(TET, POISSON):
        res = integrate_batch(desc, fek.build_batch([(unit, coeff)] * 300))
        single = integrate_element(desc, unit, coeff)
        for i in range(300):
            assert np.array_equal(res.stiffness[i], single.A)


def test_twisted_prisms_vs_refined_rule():
    z = golden("twisted_prisms.npz")
    for pb, rows in ((CONVDIFF, z["convdiff_rows"]), (POISSON, z["poisson_rows"])):
        batch = ElementBatch.from_arrays(PRISM, pb, z["geometry_rows"], rows)
        for desc in case_descriptors(PRISM, pb):
            res = integrate_batch(desc, batch)
            assert rel(res.stiffness, z[f"A_{pb.value}"]).max() < 1e-10
            assert rel(res.load, z[f"b_{pb.value}"]).max() < 1e-10


def _error_cases():
    from test_oracle import error_case_inputs

    z = golden("errors.npz")
    names = sorted({k.split("__")[0] for k in z.files if "__" in k})
    for name in names:
        geo, cof = error_case_inputs(z, name)
        et = TET if name.startswith("tet") else PRISM
        pb = POISSON if cof.shape[1] in (4, 6) else CONVDIFF
        yield z, name, et, pb, geo, cof


def test_geometry_errors_match_reference():
    import torch

    msgs = dict(line.split("\t", 1) for line in open(GOLDEN + "/error_messages.tsv").read().strip().split("\n"))
    checked = 0
    for z, name, et, pb, geo, cof in _error_cases():
        batch = ElementBatch.from_arrays(et, pb, geo, cof)
        dbatch = DeviceBatch.from_host(batch)
        for desc in case_descriptors(et, pb):
            want = tuple(int(x) for x in z[f"{name}__{desc.short_name()}"])
            for b in (batch, dbatch):
                with pytest.raises(fek.GeometryError) as err:
                    integrate_batch(desc, b)
                kind = 1 if isinstance(err.value, fek.DegenerateElement) else 2
                point = -1 if err.value.point_index is None else err.value.point_index
                assert (kind, err.value.element_index, point) == want, (name, desc.short_name())
                assert str(err.value) == msgs[f"{name}__{desc.short_name()}"]
                checked += 1
    torch.cuda.synchronize()
    assert checked >= 40


def test_geometry_errors_fp32_locate_the_same_failure():
    """fp32 kernels (the prism ones run the two zeta levels as one FFMA2 pair) locate the reference's
    failure on the golden error batches: same element always; same kind and point for inverted
    elements.  An exactly degenerate element has det J = 0 only to fp32 rounding (1e-14 diag^3 is
    below fp32 resolution), so there fp32 may report it as inverted, or at another point."""
    import torch

    checked = 0
    for z, name, et, pb, geo, cof in _error_cases():
        dbatch = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof), dtype=torch.float32)
        for desc in case_descriptors(et, pb):
            want = tuple(int(x) for x in z[f"{name}__{desc.short_name()}"])
            with pytest.raises(fek.GeometryError) as err:
                integrate_batch(desc, dbatch)
            kind = 1 if isinstance(err.value, fek.DegenerateElement) else 2
            point = -1 if err.value.point_index is None else err.value.point_index
            if want[0] == 2:
                assert (kind, err.value.element_index, point) == want, (name, desc.short_name())
            else:
                assert err.value.element_index == want[1], (name, desc.short_name())
            checked += 1
    assert checked >= 20


def test_prism_inverted_on_the_upper_level_only():
    """A prism whose top triangle is mirrored is inverted at the three upper-level points only
    (q = 1, 3, 5): the reported point is 1 in fp64 and fp32 (lane y of the fp32 level pairs),
    for every descriptor, as the oracle's first-error rule says."""
    import torch

    from oracle import numpy_oracle as O
    from paper_1504_01023_b200.verify import random_coefficients, random_prism_geometry

    rng = np.random.default_rng(77)
    et, pb = ElementType.PRISM, ProblemClass.CONV_DIFF
    elems = [(random_prism_geometry(rng), random_coefficients(pb, et, rng)) for _ in range(300)]
    coords = et.reference_vertices.copy()
    coords[[4, 5]] = coords[[5, 4]]  # mirrored top triangle: the upper points invert
    elems[137] = (fek.ElementGeometry(et, coords), elems[137][1])
    batch = fek.build_batch(elems)
    for desc in case_descriptors(et, pb):
        with pytest.raises(O.OracleGeometryError) as ref:
            O.integrate(desc.variant.value, desc.geometry_path.value, pb.value, et.value,
                        batch.geometry_rows(), batch.coefficient_rows())
        assert (ref.value.kind, ref.value.element_index, ref.value.point_index) == ("inverted", 137, 1)
        for dt in (torch.float64, torch.float32):
            with pytest.raises(fek.InvertedElement) as err:
                integrate_batch(desc, DeviceBatch.from_host(batch, dtype=dt))
            assert (err.value.element_index, err.value.point_index) == (137, 1), (desc.short_name(), dt)


def test_shape_mismatch_and_descriptor_errors():
    z, batch = corpus(TET, POISSON)
    with pytest.raises(fek.ShapeMismatch):
        integrate_batch(KernelDescriptor(Variant.QSS, GeometryPath.GEO_GENERIC, POISSON, PRISM), batch)
    with pytest.raises(ValueError):
        KernelDescriptor(Variant.QSS, GeometryPath.GEO_LINEAR, POISSON, PRISM)


def test_sharded_launches_bitwise_equal_single_launch():
    """GPU-count independence: contiguous shards with base_index == one launch."""
    import torch

    z, batch = corpus(PRISM, CONVDIFF)
    desc = case_descriptors(PRISM, CONVDIFF)[0]
    whole = integrate_batch(desc, DeviceBatch.from_host(batch))
    n = batch.n_elements
    geo, cof = z["geometry_rows"], z["coefficient_rows"]
    for shards in (2, 3, 7):
        bounds = np.linspace(0, n, shards + 1).astype(int)
        parts = []
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            sub = DeviceBatch.from_host(ElementBatch.from_arrays(PRISM, CONVDIFF, geo[lo:hi], cof[lo:hi]))
            parts.append(integrate_batch(desc, sub, base_index=int(lo)).stiffness)
        assert torch.equal(torch.cat(parts), whole.stiffness)


def test_fp32_variants_within_stated_tolerance():
    import torch

    for et, pb in CASES:
        z, batch = corpus(et, pb)
        d32 = DeviceBatch.from_host(batch, dtype=torch.float32)
        for desc in case_descriptors(et, pb):
            res = integrate_batch(desc, d32)
            assert res.stiffness.dtype == torch.float32
            A = res.stiffness.double().cpu().numpy()
            b = res.load.double().cpu().numpy()
            assert rel(A, z["A_algorithm1"]).max() < 1e-4, desc.short_name()
            assert rel(b, z["b_algorithm1"]).max() < 1e-4, desc.short_name()


@pytest.mark.parametrize("n", [0, 1, 2, 63, 64, 65, 127, 128, 129, 255, 1000, 40000])
def test_ragged_sizes_and_chunking(n):
    rng = np.random.default_rng(n)
    from oracle.numpy_oracle import integrate as oracle

    for et, pb in CASES:
        z = golden(f"corpus_{et.value}_{pb.value}.npz")
        idx = rng.integers(0, z["geometry_rows"].shape[0], size=n)
        geo, cof = z["geometry_rows"][idx], z["coefficient_rows"][idx]
        batch = ElementBatch.from_arrays(et, pb, geo, cof)
        desc = case_descriptors(et, pb)[0]
        res = integrate_batch(desc, batch)
        assert res.stiffness.shape == (n, et.n_shape, et.n_shape)
        dres = integrate_batch(desc, DeviceBatch.from_host(batch))  # device path: tile tails (64 / 128)
        assert np.array_equal(dres.stiffness.cpu().numpy(), res.stiffness)
        assert np.array_equal(dres.load.cpu().numpy(), res.load)
        if n:
            A, b = oracle(desc.variant.value, desc.geometry_path.value, pb.value, et.value, geo, cof)
            assert rel(res.stiffness, A).max() <= TOL
            assert rel(res.load, b).max() <= TOL


def test_reference_objects_cross_the_boundary_duck_typed():
    """A feklab-like descriptor/batch (enums matched by .value) is accepted."""
    from types import SimpleNamespace

    z, batch = corpus(TET, CONVDIFF)
    e = lambda v: SimpleNamespace(value=v)  # noqa: E731
    desc = SimpleNamespace(variant=e("qss"), geometry_path=e("linear"), problem=e("convdiff"), element=e("tet"))
    foreign = SimpleNamespace(element_type=e("tet"), problem=e("convdiff"), n_elements=batch.n_elements,
                              layout=SimpleNamespace(kind=e("major"), lane_width=1),
                              geometry_data=np.array(batch.geometry_data),
                              coefficient_data=np.array(batch.coefficient_data))
    res = integrate_batch(desc, foreign)
    assert rel(res.stiffness, z["A_qss_linear_tet_convdiff"]).max() <= TOL


def test_flat_output_layouts():
    z, batch = corpus(TET, POISSON)
    res = integrate_batch(case_descriptors(TET, POISSON)[0], batch)
    rows = res.output_rows()
    assert rows.shape == (batch.n_elements, 20)
    assert np.array_equal(res.flat_output(), rows.reshape(-1))
    res.out_layout = BatchLayout(LayoutKind.LANE_INTERLEAVED, 8)
    flat = res.flat_output(pad_value=0.0)
    assert np.array_equal(flat[3: 8 * 20: 8], rows[3])
    dres = integrate_batch(case_descriptors(TET, POISSON)[0], DeviceBatch.from_host(batch),
                           out_layout=BatchLayout(LayoutKind.LANE_INTERLEAVED, 8))
    assert np.array_equal(dres.flat_output(pad_value=0.0).cpu().numpy(), flat)


@pytest.mark.parametrize("et,pb", [(TET, CONVDIFF), (PRISM, CONVDIFF), (PRISM, POISSON)],
                         ids=lambda c: getattr(c, "value", c))
def test_pageable_host_batches_are_staged_bitwise(et, pb):
    """A caller's plain numpy (pageable) ElementBatch goes through fek_integrate_host_staged; the
    results equal the page-locked path's bit for bit, also for a lane-interleaved layout."""
    from paper_1504_01023_b200 import hostmem, mesh
    from paper_1504_01023_b200.kernels import batched as KB
    from paper_1504_01023_b200.layout import convert

    spec = mesh.spec_for_element_count(et, 700_000)
    geo = mesh.geometry_rows(spec)
    cof = mesh.coefficient_rows(spec.n_elements, pb, et, 3)
    pinned = ElementBatch.from_arrays(et, pb, geo, cof)
    assert hostmem.is_pinned(pinned.geometry_data)
    for batch in (pinned, convert(pinned, BatchLayout(LayoutKind.LANE_INTERLEAVED, 16))):
        plain = ElementBatch(batch.element_type, batch.problem, batch.n_elements, batch.layout,
                             np.array(batch.geometry_data), np.array(batch.coefficient_data))
        assert not hostmem.is_pinned(plain.geometry_data) and KB._needs_staging(plain.geometry_data)
        desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
        want, got = integrate_batch(desc, batch), integrate_batch(desc, plain)
        assert np.array_equal(want.stiffness, got.stiffness) and np.array_equal(want.load, got.load)


def test_staged_abi_with_pageable_outputs():
    """fek_integrate_host_staged also stages PAGEABLE outputs (a C caller's malloc'd A / b)."""
    import ctypes

    import torch

    from paper_1504_01023_b200 import _native, hostmem, mesh
    from paper_1504_01023_b200.kernels.batched import _desc_struct, _host_streams
    from paper_1504_01023_b200.layout import ELEMENT_MAJOR

    et, pb = PRISM, CONVDIFF
    spec = mesh.spec_for_element_count(et, 300_000)
    geo = np.ascontiguousarray(mesh.geometry_rows(spec).reshape(-1))
    cof = np.ascontiguousarray(mesh.coefficient_rows(spec.n_elements, pb, et, 4).reshape(-1))
    n = spec.n_elements
    A, b = np.empty((n, 6, 6)), np.empty((n, 6))
    assert not hostmem.is_pinned(A)
    lib = _native.load()
    desc = KernelDescriptor(Variant.QSS, GeometryPath.GEO_GENERIC, pb, et)
    dd = _desc_struct(desc, ELEMENT_MAJOR, n, 0, 0, geo.ctypes.data, cof.ctypes.data, A.ctypes.data, b.ctypes.data, 0)
    streams = _host_streams(torch.cuda.current_device())
    handles = (ctypes.c_void_p * len(streams))(*[s.cuda_stream for s in streams])
    chunk = 65536
    ws_bytes = lib.fek_host_workspace_bytes(ctypes.byref(dd), len(streams), chunk)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    st_bytes = lib.fek_host_staging_bytes(ctypes.byref(dd), len(streams), chunk)
    staging = hostmem.empty(-(-st_bytes // 8), pin=True)
    torch.cuda.synchronize()
    key = ctypes.c_ulonglong()
    rc = lib.fek_integrate_host_staged(ctypes.byref(dd), ws.data_ptr(), ws_bytes, len(streams), handles, chunk,
                                       staging.ctypes.data, st_bytes, 4, ctypes.byref(key))
    assert rc == 0 and key.value == _native.NO_ERROR
    ref = integrate_batch(desc, ElementBatch.from_arrays(et, pb, geo.reshape(n, -1), cof.reshape(n, -1)))
    assert np.array_equal(A, ref.stiffness) and np.array_equal(b, ref.load)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("et,pb", CASES, ids=lambda c: getattr(c, "value", c))
def test_tile_and_cta_variants_are_bitwise_identical(et, pb, dtype):
    """The tuner's launch knobs (tile T = 64/128/256 instantiations, CTAs/SM caps) never change a
    result: every element runs one instruction sequence whatever the launch shape."""
    import torch

    from paper_1504_01023_b200 import mesh

    spec = mesh.spec_for_element_count(et, 20_000)
    geo = mesh.geometry_rows(spec)
    if et is PRISM:
        geo = mesh.jitter_top_faces(geo, spec, seed=5)
    cof = mesh.coefficient_rows(spec.n_elements, pb, et, 5)
    dev = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof), dtype=getattr(torch, dtype))
    desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
    want = integrate_batch(desc, dev)
    for tile in (64, 128, 256):
        for ctas in (0, 1, 2):
            got = integrate_batch(desc, dev, tile=tile, ctas_per_sm=ctas)
            assert torch.equal(got.stiffness, want.stiffness) and torch.equal(got.load, want.load), (tile, ctas)
    with pytest.raises(fek.NativeLibraryError):
        integrate_batch(KernelDescriptor(Variant.SQS, fek.natural_path(et), pb, et), dev, tile=128)


def test_out_arrays_are_validated_before_the_launch():
    """integrate_batch(..., out=(A, b)) rejects wrong dtype / shape / device / strides / alignment
    instead of letting the kernel write through raw pointers."""
    import torch

    z, host = corpus(PRISM, CONVDIFF)
    dev = DeviceBatch.from_host(host)
    n = dev.n_elements
    desc = KernelDescriptor(Variant.QSS, GeometryPath.GEO_GENERIC, CONVDIFF, PRISM)
    ok = (torch.empty((n, 6, 6), dtype=torch.float64, device="cuda"), torch.empty((n, 6), dtype=torch.float64,
                                                                                    device="cuda"))
    integrate_batch(desc, dev, out=ok)
    bad = [
        (torch.empty((n, 6, 6), dtype=torch.float32, device="cuda"), ok[1]),          # dtype
        (torch.empty((n - 1, 6, 6), dtype=torch.float64, device="cuda"), ok[1]),      # shape
        (ok[0], torch.empty((n, 6), dtype=torch.float64)),                            # host tensor
        (torch.empty((n, 6, 12), dtype=torch.float64, device="cuda")[:, :, :6], ok[1]),  # strided
        (torch.empty(n * 36 + 1, dtype=torch.float64, device="cuda")[1:].view(n, 6, 6), ok[1]),  # misaligned
    ]
    for out in bad:
        with pytest.raises((TypeError, ValueError)):
            integrate_batch(desc, dev, out=out)
    with pytest.raises(ValueError):
        integrate_batch(desc, dev, out=ok, packed=True)
    with pytest.raises(TypeError):
        integrate_batch(desc, host, out=ok)


def test_concurrent_host_calls_from_two_threads():
    """integrate_batch is re-entrant (batched.py's contract): two host threads integrating different
    host batches at once (own streams and staging per thread) get the sequential results bitwise."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1504_01023_b200 import mesh

    jobs = []
    for et, pb, k in ((TET, CONVDIFF, 1), (PRISM, CONVDIFF, 2), (PRISM, POISSON, 3)):
        spec = mesh.spec_for_element_count(et, 600_000)
        geo = mesh.geometry_rows(spec)
        cof = mesh.coefficient_rows(spec.n_elements, pb, et, k)
        batch = ElementBatch.from_arrays(et, pb, geo, cof)
        plain = ElementBatch(et, pb, batch.n_elements, batch.layout, np.array(batch.geometry_data),
                             np.array(batch.coefficient_data))  # pageable: the staged path
        desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
        jobs += [(desc, batch), (desc, plain)]
    want = [integrate_batch(d, b) for d, b in jobs]
    with ThreadPoolExecutor(3) as ex:
        got = list(ex.map(lambda j: integrate_batch(*j), jobs))
    for w, g in zip(want, got):
        assert np.array_equal(w.stiffness, g.stiffness) and np.array_equal(w.load, g.load)
