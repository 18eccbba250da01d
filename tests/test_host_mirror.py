"""Host-side mirror of the reference API: constants, layouts, descriptors, counts, meshes.

CPU only.  The reference-element tables and synthetic meshes must be
bit-identical to the reference's (golden files generated from it).
"""

import os

import numpy as np
import pytest

import paper_1504_01023_b200 as fek
from conftest import golden
from paper_1504_01023_b200 import (BatchLayout, CoefficientSet, ElementBatch, ElementGeometry, ElementType,
                                   GeometryPath, KernelDescriptor, LayoutKind, ProblemClass, Variant, mesh)
from paper_1504_01023_b200.kernels.counts import OP_TOTALS, phase_op_counts

TET, PRISM = ElementType.TETRAHEDRON, ElementType.PRISM


def test_reference_element_tables_bitwise():
    r = golden("refelem.npz")
    for et in ElementType:
        rule, table = fek.reference_element(et)
        assert np.array_equal(rule.points, r[f"{et.value}_points"])
        assert np.array_equal(rule.weights, r[f"{et.value}_weights"])
        assert np.array_equal(table.values, r[f"{et.value}_values"])
        assert np.array_equal(table.local_derivatives, r[f"{et.value}_local_derivatives"])
        assert not table.values.flags.writeable


def test_shape_at_rejects_outside_points():
    with pytest.raises(ValueError):
        fek.shape_at(TET, [0.5, 0.5, 0.5])
    with pytest.raises(ValueError):
        fek.shape_at(PRISM, [0.2, 0.2, 1.5])
    vals, ders = fek.shape_at(PRISM, [0.2, 0.3, 0.1])
    assert abs(vals.sum() - 1.0) < 1e-14 and np.abs(ders.sum(axis=0)).max() < 1e-14


def test_descriptors():
    assert len(fek.all_descriptors()) == 18
    assert len(fek.case_descriptors(TET, ProblemClass.POISSON)) == 6
    assert len(fek.case_descriptors(PRISM, ProblemClass.CONV_DIFF)) == 3
    with pytest.raises(ValueError):
        KernelDescriptor(Variant.QSS, GeometryPath.GEO_LINEAR, ProblemClass.POISSON, PRISM)
    d = KernelDescriptor(Variant.SQS, GeometryPath.GEO_GENERIC, ProblemClass.CONV_DIFF, TET)
    assert d.short_name() == "sqs_generic_tet_convdiff"


def test_counts_match_table4():
    assert fek.global_accesses(TET, ProblemClass.POISSON) == 36
    assert fek.global_accesses(PRISM, ProblemClass.POISSON) == 66
    assert fek.global_accesses(TET, ProblemClass.CONV_DIFF) == 52
    assert fek.global_accesses(PRISM, ProblemClass.CONV_DIFF) == 80
    for (v, e, p), total in OP_TOTALS.items():
        c = phase_op_counts(KernelDescriptor(v, GeometryPath.GEO_GENERIC, p, e))
        assert c.total == total
        assert min(c.geo_derivs, c.jacobian_terms, c.shape_derivs, c.final_update) > 0
        assert c.geo_derivs + c.jacobian_terms + c.shape_derivs + c.final_update == total


def test_interleaved_index_formula_and_padding(rng):
    rows = rng.uniform(size=(6, 12))
    flat = fek.pack_rows(rows, BatchLayout(LayoutKind.LANE_INTERLEAVED, 4))
    assert flat.shape == (fek.flat_length(6, 12, BatchLayout(LayoutKind.LANE_INTERLEAVED, 4)),)
    for e in range(6):
        for d in range(12):
            assert flat[(e // 4) * 4 * 12 + d * 4 + e % 4] == rows[e, d]
    assert np.isnan(flat).sum() == 2 * 12


@pytest.mark.parametrize("w", [1, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("n", [1, 5, 63, 64, 65, 200])
def test_pack_unpack_round_trip(w, n, rng):
    rows = rng.uniform(size=(n, 7))
    layout = BatchLayout(LayoutKind.LANE_INTERLEAVED, w)
    assert np.array_equal(fek.unpack_rows(fek.pack_rows(rows, layout), n, 7, layout), rows)


def test_lane_width_validated():
    with pytest.raises(ValueError):
        BatchLayout(LayoutKind.LANE_INTERLEAVED, 3)


def test_build_extract_convert(rng):
    els = []
    for _ in range(11):
        g = ElementGeometry(TET, rng.uniform(size=(4, 3)))
        els.append((g, CoefficientSet.convdiff(rng.uniform(size=(4, 4)), rng.uniform(size=4))))
    for layout in (fek.ELEMENT_MAJOR, BatchLayout(LayoutKind.LANE_INTERLEAVED, 4),
                   BatchLayout(LayoutKind.LANE_INTERLEAVED, 64)):
        b = fek.build_batch(els, layout)
        for e, (g, c) in enumerate(els):
            g2, c2 = fek.extract(b, e)
            assert np.array_equal(g2.coords, g.coords) and np.array_equal(c2.flat(), c.flat())
        back = fek.convert(b, fek.ELEMENT_MAJOR)
        assert np.array_equal(back.geometry_rows(), fek.build_batch(els).geometry_rows())
    with pytest.raises(fek.HeterogeneousBatch):
        fek.build_batch([els[0], (ElementGeometry(PRISM, rng.uniform(size=(6, 3))), els[0][1])])


def test_fekb_file_round_trip(tmp_path, rng):
    rows = rng.uniform(size=(9, 12))
    cof = rng.uniform(size=(9, 4))
    b = ElementBatch.from_arrays(TET, ProblemClass.POISSON, rows, cof, BatchLayout(LayoutKind.LANE_INTERLEAVED, 4),
                                 pad_value=0.0)
    path = tmp_path / "b.fekb"
    fek.write_batch(b, path)
    assert os.path.getsize(path) == 32 + 8 * (b.geometry_data.size + b.coefficient_data.size)
    c = fek.read_batch(path)
    assert c.layout == b.layout and c.n_elements == 9
    assert np.array_equal(c.geometry_data, b.geometry_data)
    raw = path.read_bytes()
    (tmp_path / "bad.fekb").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="magic"):
        fek.read_batch(tmp_path / "bad.fekb")
    (tmp_path / "short.fekb").write_bytes(raw[:-8])
    with pytest.raises(ValueError, match="truncated"):
        fek.read_batch(tmp_path / "short.fekb")


def test_meshes_bitwise_equal_reference():
    z = golden("meshes.npz")
    for name in ("tet_432", "tet_222", "prism_53", "prism_44"):
        nx, ny, nz, seed = (int(v) for v in z[name + "_spec"])
        et = TET if name.startswith("tet") else PRISM
        pb = ProblemClass.CONV_DIFF if z[name + "_coefficient_rows"].shape[1] == 20 else ProblemClass.POISSON
        b = mesh.generate_mesh(mesh.MeshSpec(nx, ny, nz, et), seed, pb)
        assert np.array_equal(b.geometry_rows(), z[name + "_geometry_rows"])
        assert np.array_equal(b.coefficient_rows(), z[name + "_coefficient_rows"])


def test_bench_config_sizes():
    c = mesh.bench_configs()
    assert c["C1"].spec.n_elements == 1_053_696
    assert c["C2"].spec.n_elements == 4_088_832
    assert c["C3"].spec.n_elements == 4_004_450
    assert c["C4"].spec.n_elements == 16_006_482
    assert c["C5T"].spec.n_elements + c["C5P"].spec.n_elements == 64_156_250


def test_jittered_prisms_stay_valid():
    from oracle import numpy_oracle as O

    spec = mesh.MeshSpec(40, 30, 1, PRISM)
    geo = mesh.jitter_top_faces(mesh.geometry_rows(spec), spec, seed=1)
    assert not np.array_equal(geo, mesh.geometry_rows(spec))
    A, _ = O.integrate("qss", "generic", "poisson", "prism", geo, np.ones((spec.n_elements, 6)))
    assert np.isfinite(A).all()  # no degenerate/inverted element raised


def test_duck_typed_descriptor_coercion():
    from types import SimpleNamespace

    from paper_1504_01023_b200.problems import coerce_descriptor

    e = lambda v: SimpleNamespace(value=v)  # noqa: E731
    d = coerce_descriptor(SimpleNamespace(variant=e("ssq"), geometry_path=e("generic"), problem=e("poisson"),
                                          element=e("prism")))
    assert d == KernelDescriptor(Variant.SSQ, GeometryPath.GEO_GENERIC, ProblemClass.POISSON, PRISM)
    with pytest.raises(TypeError):
        coerce_descriptor(SimpleNamespace(variant=e("xyz"), geometry_path=e("generic"), problem=e("poisson"),
                                          element=e("prism")))


@pytest.mark.parametrize("key", ["C1", "C2", "C3"])
def test_bench_inputs_equal_reference_generator(key):
    """Host restatement of the benchmark inputs == the reference's generate_mesh (sampled, full size)."""
    z = golden(f"bench_{key}.npz")
    cfg = mesh.bench_configs()[key]
    geo, cof = mesh.config_rows(cfg)
    assert geo.shape[0] == int(z["n_elements"][0])
    assert np.array_equal(geo[z["index"]], z["geometry_rows"])
    assert np.array_equal(cof[z["index"]], z["coefficient_rows"])


@pytest.mark.parametrize("et", [ElementType.TETRAHEDRON, ElementType.PRISM])
def test_element_nodes_are_consistent_with_the_geometry(et):
    """mesh.element_nodes: one coordinate per node number across all elements, every node used."""
    from paper_1504_01023_b200 import mesh

    spec = mesh.MeshSpec(4, 3, 5, et) if et is ElementType.TETRAHEDRON else mesh.MeshSpec(7, 5, 1, et)
    nodes = mesh.element_nodes(spec)
    geo = mesh.geometry_rows(spec).reshape(len(nodes), -1, 3)
    assert nodes.dtype == np.int32 and nodes.shape == (spec.n_elements, et.n_vertices)
    coords = np.full((mesh.node_count(spec), 3), np.nan)
    coords[nodes.reshape(-1)] = geo.reshape(-1, 3)
    # (a node reached from different cells differs by rounding only: x0 + h vs (i + 1) h)
    assert np.allclose(coords[nodes], geo, rtol=0, atol=1e-14) and not np.isnan(coords).any()


def test_config_window_is_the_prefix_of_the_full_configuration():
    from paper_1504_01023_b200 import mesh

    for key in ("C1", "C3"):
        cfg = mesh.bench_configs()[key]
        g, c = mesh.config_rows(cfg)
        gw, cw = mesh.config_window(cfg, 50_001)
        assert np.array_equal(g[:50_001], gw) and np.array_equal(c[:50_001], cw)


def test_bind_exception_types_makes_the_boundary_raise_host_classes():
    """errors.bind_exception_types(feklab.errors): the drop-in raises the host package's classes
    (looked up at raise time by kernels/batched.py, kernels/scalar.py and geometry.py)."""
    import types

    from paper_1504_01023_b200 import errors
    from paper_1504_01023_b200.kernels import batched

    saved = {n: getattr(errors, n) for n in errors.BOUNDARY_TYPES}

    class HostGeometryError(Exception):
        def __init__(self, message, element_index=None, point_index=None):
            super().__init__(message)
            self.element_index, self.point_index = element_index, point_index

    host = types.SimpleNamespace(GeometryError=HostGeometryError,
                                 DegenerateElement=type("DegenerateElement", (HostGeometryError,), {}),
                                 InvertedElement=type("InvertedElement", (HostGeometryError,), {}),
                                 ShapeMismatch=type("ShapeMismatch", (Exception,), {}))
    try:
        errors.bind_exception_types(host)
        with pytest.raises(host.InvertedElement) as err:
            batched._raise_geometry((17, 3, 2), lambda e, q: (-0.5, 1e-14))
        assert (err.value.element_index, err.value.point_index) == (17, 3)
        assert "det J = -5.000e-01 < 0" in str(err.value)
    finally:
        for n, cls in saved.items():
            setattr(errors, n, cls)
    with pytest.raises(fek.InvertedElement):
        batched._raise_geometry((17, 3, 2), lambda e, q: (-0.5, 1e-14))


def test_first_pattern_miss_on_cpu():
    """The rare-path pattern check of assemble_batch (torch; runs on CPU tensors too)."""
    import torch

    from paper_1504_01023_b200 import mesh
    from paper_1504_01023_b200.kernels.apply import _first_pattern_miss, csr_pattern

    spec = mesh.MeshSpec(4, 3, 2, mesh.ElementType.TETRAHEDRON)
    nodes = torch.from_numpy(mesh.element_nodes(spec))
    nn = mesh.node_count(spec)
    row_ptr, col = csr_pattern(nodes, nn)
    assert _first_pattern_miss(nodes, row_ptr, col) is None
    rp, cl = row_ptr.long(), col.clone()
    i, j = int(nodes[7, 0]), int(nodes[7, 3])
    k = int(rp[i]) + int(torch.searchsorted(cl[rp[i]:rp[i + 1]].contiguous(), j))
    cl = torch.cat([cl[:k], cl[k + 1:]])
    rp[i + 1:] -= 1
    first = min(e for e in range(len(nodes)) if i in nodes[e].tolist() and j in nodes[e].tolist())
    assert _first_pattern_miss(nodes, rp.int(), cl) == first
