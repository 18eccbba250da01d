"""Fused matrix-free apply (fek_apply, kernels/apply.py) against the oracle and the two-pass path.

y = sum_e P_e^T A_e P_e x and f = sum_e P_e^T b_e, with A_e, b_e kept in the integration kernel's
registers.  The element matrices are the reference's (oracle: bitwise-pinned numpy restatement);
only the order of the atomicAdd accumulation differs, so entries are compared relative to the
sum of the magnitudes of their contributions (<= 1e-13).
"""

import numpy as np
import pytest
import torch

import paper_1504_01023_b200 as fek
from oracle import numpy_oracle as O
from paper_1504_01023_b200 import DeviceBatch, ElementBatch, ElementType, KernelDescriptor, ProblemClass, Variant, mesh

pytestmark = pytest.mark.gpu

CASES = [(ElementType.TETRAHEDRON, ProblemClass.CONV_DIFF, mesh.MeshSpec(12, 10, 9, ElementType.TETRAHEDRON)),
         (ElementType.TETRAHEDRON, ProblemClass.POISSON, mesh.MeshSpec(9, 8, 7, ElementType.TETRAHEDRON)),
         (ElementType.PRISM, ProblemClass.CONV_DIFF, mesh.MeshSpec(101, 77, 1, ElementType.PRISM)),
         (ElementType.PRISM, ProblemClass.POISSON, mesh.MeshSpec(61, 53, 1, ElementType.PRISM))]


def _setup(et, pb, spec, seed=3):
    geo = mesh.geometry_rows(spec)
    if et is ElementType.PRISM:
        geo = mesh.jitter_top_faces(geo, spec, seed=seed)
    cof = mesh.coefficient_rows(spec.n_elements, pb, et, seed)
    nodes = mesh.element_nodes(spec)
    x = np.random.default_rng(seed).uniform(-1, 1, mesh.node_count(spec))
    return geo, cof, nodes, x


def _scatter(A, b, nodes, x, n_nodes):
    xe = x[nodes]                                       # (n, ns)
    ye = np.einsum("ers,es->er", A, xe)
    mag = np.einsum("ers,es->er", np.abs(A), np.abs(xe))
    y, f, ym, fm = (np.zeros(n_nodes) for _ in range(4))
    np.add.at(y, nodes, ye)
    np.add.at(ym, nodes, mag)
    np.add.at(f, nodes, b)
    np.add.at(fm, nodes, np.abs(b))
    return y, f, ym, fm


@pytest.mark.parametrize("et,pb,spec", CASES, ids=lambda c: getattr(c, "value", None) or str(getattr(c, "nx", c)))
def test_apply_matches_oracle(et, pb, spec):
    geo, cof, nodes, x = _setup(et, pb, spec)
    desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
    A, b = O.integrate("qss", desc.geometry_path.value, pb.value, et.value, geo, cof)
    y_ref, f_ref, ym, fm = _scatter(A, b, nodes, x, len(x))
    dev = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof))
    y, f = fek.apply_batch(desc, dev, torch.from_numpy(nodes).cuda(), torch.from_numpy(x).cuda())
    y, f = y.cpu().numpy(), f.cpu().numpy()
    assert (np.abs(y - y_ref) <= 1e-13 * ym + 1e-300).all()
    assert (np.abs(f - f_ref) <= 1e-13 * fm + 1e-300).all()


def test_apply_equals_two_pass_at_c4_size():
    """C4 (16M jittered prisms, ConvDiff): fused apply vs integrate_batch -> stored A, b -> scatter."""
    cfg = mesh.bench_configs()["C4"]
    geo, cof = mesh.device_config(cfg)
    et, pb = cfg.spec.element_type, cfg.problem
    n = cfg.spec.n_elements
    dev = DeviceBatch(et, pb, n, fek.ELEMENT_MAJOR, geo, cof)
    nodes = torch.from_numpy(mesh.element_nodes(cfg.spec)).cuda()
    x = torch.rand(mesh.node_count(cfg.spec), dtype=torch.float64, device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(7)) * 2 - 1
    desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
    y, f = fek.apply_batch(desc, dev, nodes, x)
    res = fek.integrate_batch(desc, dev)
    idx = nodes.long()
    xe = x[idx]
    ye = torch.einsum("ers,es->er", res.stiffness, xe)
    mag = torch.einsum("ers,es->er", res.stiffness.abs(), xe.abs())
    y2, ym, f2, fm = (torch.zeros_like(x) for _ in range(4))
    y2.index_add_(0, idx.reshape(-1), ye.reshape(-1))
    ym.index_add_(0, idx.reshape(-1), mag.reshape(-1))
    f2.index_add_(0, idx.reshape(-1), res.load.reshape(-1))
    fm.index_add_(0, idx.reshape(-1), res.load.abs().reshape(-1))
    assert bool(((y - y2).abs() <= 1e-13 * ym).all()) and bool(((f - f2).abs() <= 1e-13 * fm).all())


def test_apply_reports_geometry_errors_like_integrate_batch():
    et, pb, spec = CASES[2]
    geo, cof, nodes, x = _setup(et, pb, spec)
    geo[1234] = -geo[1234]
    dev = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof))
    desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
    with pytest.raises(fek.InvertedElement) as err:
        fek.apply_batch(desc, dev, torch.from_numpy(nodes).cuda(), torch.from_numpy(x).cuda())
    assert (err.value.element_index, err.value.point_index) == (1234, 0)
    with pytest.raises(fek.NativeLibraryError):
        fek.apply_batch(KernelDescriptor(Variant.SQS, fek.natural_path(et), pb, et), dev,
                        torch.from_numpy(nodes).cuda(), torch.from_numpy(x).cuda())


def test_apply_rejects_out_of_range_nodes():
    et, pb, spec = CASES[0]
    geo, cof, nodes, x = _setup(et, pb, spec)
    dev = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof))
    desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
    bad = nodes.copy()
    bad[5, 2] = len(x)
    with pytest.raises(ValueError):
        fek.apply_batch(desc, dev, torch.from_numpy(bad).cuda(), torch.from_numpy(x).cuda())


@pytest.mark.parametrize("et,pb,spec", CASES, ids=lambda c: getattr(c, "value", None) or str(getattr(c, "nx", c)))
def test_assemble_matches_oracle(et, pb, spec):
    """CSR assembly fused with the integration: every stored entry within 1e-13 of the sum of its
    contributions' magnitudes against the oracle's matrices summed per node pair on the host."""
    geo, cof, nodes, x = _setup(et, pb, spec)
    desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
    A, b = O.integrate("qss", desc.geometry_path.value, pb.value, et.value, geo, cof)
    nn = len(x)
    dev = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof))
    tn = torch.from_numpy(nodes).cuda()
    row_ptr, col = fek.csr_pattern(tn, nn)
    values, f = fek.assemble_batch(desc, dev, tn, row_ptr, col)
    rp, cl = row_ptr.cpu().numpy(), col.cpu().numpy()
    assert (np.diff(rp) > 0).all() and all((np.diff(cl[rp[i]:rp[i + 1]]) > 0).all() for i in range(0, nn, 97))
    rows = np.repeat(np.arange(nn), np.diff(rp))
    keys = rows.astype(np.int64) * nn + cl
    pr = np.repeat(nodes[:, :, None], nodes.shape[1], 2).reshape(-1).astype(np.int64)
    pc = np.repeat(nodes[:, None, :], nodes.shape[1], 1).reshape(-1).astype(np.int64)
    pos = np.searchsorted(keys, pr * nn + pc)
    ref, mag = np.zeros(len(cl)), np.zeros(len(cl))
    np.add.at(ref, pos, A.reshape(-1))
    # scale: each contribution's element-matrix magnitude (entries that vanish exactly in the
    # reference's arithmetic come out at rounding level in the kernel's)
    np.add.at(mag, pos, np.repeat(np.abs(A).reshape(len(A), -1).max(1), A.shape[1] * A.shape[2]))
    got = values.cpu().numpy()
    assert (np.abs(got - ref) <= 1e-13 * mag + 1e-300).all()
    y_ref, f_ref, _, fm = _scatter(A, b, nodes, x, nn)
    assert (np.abs(f.cpu().numpy() - f_ref) <= 1e-13 * fm + 1e-300).all()
    # the assembled matrix applied to x equals the fused apply
    y, _ = fek.apply_batch(desc, dev, tn, torch.from_numpy(x).cuda(), f=False)
    csr = torch.sparse_csr_tensor(row_ptr.long(), col.long(), values, size=(nn, nn))
    y2 = (csr @ torch.from_numpy(x).cuda().unsqueeze(1)).squeeze(1)
    _, _, ym, _ = _scatter(A, b, nodes, x, nn)
    assert bool(((y - y2).abs().cpu() <= torch.from_numpy(2e-13 * ym + 1e-300)).all())


@pytest.mark.parametrize("et,pb,spec", CASES[::2], ids=lambda c: getattr(c, "value", None) or str(getattr(c, "nx", c)))
def test_assemble_reports_pattern_miss(et, pb, spec):
    """A pattern lacking one node pair: the kernel skips that contribution (no write elsewhere) and
    assemble_batch raises naming the first element that needs it; malformed structures are rejected."""
    geo, cof, nodes, x = _setup(et, pb, spec)
    desc = KernelDescriptor(Variant.QSS, fek.natural_path(et), pb, et)
    nn = len(x)
    dev = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof))
    tn = torch.from_numpy(nodes).cuda()
    row_ptr, col = fek.csr_pattern(tn, nn)
    rp, cl = row_ptr.cpu().numpy().astype(np.int64), col.cpu().numpy()
    # drop the pair (i, j) of element 57's rows 1 and 2 from row i
    i, j = int(nodes[57, 1]), int(nodes[57, 2])
    k = rp[i] + int(np.searchsorted(cl[rp[i]:rp[i + 1]], j))
    assert cl[k] == j
    cl2 = np.delete(cl, k)
    rp2 = rp.copy()
    rp2[i + 1:] -= 1
    first = min(e for e in range(len(nodes)) if i in nodes[e] and j in nodes[e])
    values = torch.full((len(cl2),), 0.0, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match=f"element {first}"):
        fek.assemble_batch(desc, dev, tn, torch.from_numpy(rp2.astype(np.int32)).cuda(),
                           torch.from_numpy(cl2).cuda(), values)
    # the entries that remain match a full assembly's (nothing landed in a neighbour's slot)
    full, _ = fek.assemble_batch(desc, dev, tn, row_ptr, col)
    keep = np.ones(len(cl), bool)
    keep[k] = False
    got, ref = values.cpu().numpy(), full.cpu().numpy()[keep]
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    # malformed structures
    bad = rp.astype(np.int32).copy()
    bad[-1] -= 1
    with pytest.raises(ValueError, match="row_ptr"):
        fek.assemble_batch(desc, dev, tn, torch.from_numpy(bad).cuda(), col)
    badc = cl.copy()
    badc[3] = nn
    with pytest.raises(ValueError, match="col"):
        fek.assemble_batch(desc, dev, tn, row_ptr, torch.from_numpy(badc).cuda())
