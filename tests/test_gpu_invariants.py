"""Structural invariants of the integrals on the GPU (test_acceptance.py:205-282 restated).

1000-element seeded corpora per element type (random well-shaped tets,
randomly mapped + jittered prisms), run through the device path:
* row-sum nullity: derivative-only coefficients annihilate constants;
* symmetry: symmetric derivative block + reaction term -> symmetric A;
* affine scaling laws on tets: pure diffusion ~ h, pure reaction ~ h^3;
* Poisson = ConvDiff with identity diffusion and the load folded into d0
  (cross-problem consistency on the same geometry).
"""

import numpy as np
import pytest

from oracle import numpy_oracle as O
from paper_1504_01023_b200 import (DeviceBatch, ElementBatch, ElementType, GeometryPath, KernelDescriptor,
                                   ProblemClass, Variant, integrate_batch)

pytestmark = pytest.mark.gpu

TET, PRISM = ElementType.TETRAHEDRON, ElementType.PRISM
CD, PO = ProblemClass.CONV_DIFF, ProblemClass.POISSON
N = 1000


def random_geometry(et, rng, n):
    if et is TET:
        v0 = rng.uniform(-1, 1, (n, 1, 3))
        edges = rng.uniform(-1, 1, (n, 3, 3))
        det = np.linalg.det(edges)
        edges[det < 0] = edges[det < 0][:, [0, 2, 1]]
        keep = np.abs(det) > 0.05
        return np.concatenate([v0, v0 + edges], axis=1)[keep].reshape(-1, 12)
    ref = np.array([(0, 0, -1), (1, 0, -1), (0, 1, -1), (0, 0, 1), (1, 0, 1), (0, 1, 1)], dtype=float)
    lin = rng.uniform(-1, 1, (n, 3, 3)) + 2 * np.eye(3)
    shift = rng.uniform(-1, 1, (n, 1, 3))
    coords = ref @ np.transpose(lin, (0, 2, 1)) + shift + 0.05 * rng.uniform(-1, 1, (n, 6, 3))
    keep = np.linalg.det(lin) > 1.0  # well inside the valid (positively oriented) set
    return coords[keep].reshape(-1, 18)


def run(et, pb, geo, cof, variant=Variant.QSS, path=None):
    path = path or (GeometryPath.GEO_LINEAR if et is TET else GeometryPath.GEO_GENERIC)
    batch = DeviceBatch.from_host(ElementBatch.from_arrays(et, pb, geo, cof))
    res = integrate_batch(KernelDescriptor(variant, path, pb, et), batch)
    return res.stiffness.cpu().numpy(), res.load.cpu().numpy()


@pytest.mark.parametrize("et", [TET, PRISM])
def test_row_sum_nullity_and_symmetry(et):
    rng = np.random.default_rng(987654323)
    geo = random_geometry(et, rng, N)
    n = geo.shape[0]
    c = np.zeros((n, 4, 4))
    c[:, 1:, 1:] = rng.uniform(-1, 1, (n, 3, 3))
    cof = np.zeros((n, 20))
    cof[:, :16] = c.reshape(n, 16)
    for v in Variant:
        A, _ = run(et, CD, geo, cof, v, GeometryPath.GEO_GENERIC)
        norms = np.sqrt((A ** 2).sum(axis=(1, 2)))
        assert (np.abs(A.sum(axis=2)).max(axis=1) <= 1e-12 * norms).all(), v
    sym = c[:, 1:, 1:] + np.transpose(c[:, 1:, 1:], (0, 2, 1))
    c2 = np.zeros((n, 4, 4))
    c2[:, 1:, 1:] = sym
    c2[:, 0, 0] = rng.uniform(-1, 1, n)
    cof2 = np.zeros((n, 20))
    cof2[:, :16] = c2.reshape(n, 16)
    cof2[:, 16:] = rng.uniform(-1, 1, (n, 4))
    A, _ = run(et, CD, geo, cof2)
    assert O.rel_frobenius(A, np.transpose(A, (0, 2, 1))).max() < 1e-12


def test_affine_scaling_laws_tets():
    rng = np.random.default_rng(987654324)
    geo = random_geometry(TET, rng, N)
    n = geo.shape[0]
    h = 1.7
    for block, power in (("diffusion", 1.0), ("reaction", 3.0)):
        c = np.zeros((4, 4))
        if block == "diffusion":
            c[1:, 1:] = np.eye(3)
        else:
            c[0, 0] = 1.0
        cof = np.tile(np.concatenate([c.reshape(-1), np.zeros(4)]), (n, 1))
        small, _ = run(TET, CD, geo, cof)
        big, _ = run(TET, CD, geo * h, cof)
        assert O.rel_frobenius(big, h ** power * small).max() < 1e-12


@pytest.mark.parametrize("et", [TET, PRISM])
def test_poisson_equals_identity_diffusion_convdiff(et):
    rng = np.random.default_rng(987654325)
    geo = random_geometry(et, rng, N)
    n = geo.shape[0]
    c = np.zeros((4, 4))
    c[1:, 1:] = np.eye(3)
    cof_cd = np.tile(np.concatenate([c.reshape(-1), np.zeros(4)]), (n, 1))
    A_cd, _ = run(et, CD, geo, cof_cd)
    A_po, b_po = run(et, PO, geo, np.zeros((n, et.n_quad)))
    assert O.rel_frobenius(A_po, A_cd).max() < 1e-12
    assert np.all(b_po == 0.0)
    # a constant right-hand side d0 = 1 equals ConvDiff with d = (1, 0, 0, 0)
    cof_cd[:, 16] = 1.0
    _, b_cd = run(et, CD, geo, cof_cd)
    _, b_po1 = run(et, PO, geo, np.ones((n, et.n_quad)))
    assert O.rel_frobenius(b_po1, b_cd).max() < 1e-12
