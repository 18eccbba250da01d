"""Per-element Jacobians on the GPU (``fek_jacobian``), restating ``pkg/tests/test_geometry.py``.

``jacobian_affine`` / ``jacobian_at_point`` return the reference's
``JacobianData`` computed by the library's own Jacobian arithmetic; the
expectations and tolerances are the reference test's.
"""

import numpy as np
import pytest

from paper_1504_01023_b200 import DegenerateElement, ElementGeometry, ElementType, InvertedElement, reference_element
from paper_1504_01023_b200.geometry import global_derivatives, jacobian_affine, jacobian_at_point
from paper_1504_01023_b200.verify import random_prism_geometry, random_tet_geometry

pytestmark = pytest.mark.gpu

TET, PRISM = ElementType.TETRAHEDRON, ElementType.PRISM


def test_identity_and_scaled_tet():
    rule, table = reference_element(TET)
    jac = jacobian_affine(ElementGeometry(TET, TET.reference_vertices), rule)
    assert np.abs(jac.dx_dxi - np.eye(3)).max() < 1e-15
    assert abs(jac.det - 1.0) < 1e-15 and abs(jac.vol.sum() - 1.0 / 6.0) < 1e-15
    gdx = global_derivatives(jac, table.local_derivatives[0])
    assert np.abs(gdx - table.local_derivatives[0]).max() < 1e-15
    jac = jacobian_affine(ElementGeometry(TET, 2.0 * TET.reference_vertices), rule)
    assert abs(jac.det - 8.0) < 1e-14 and abs(jac.vol.sum() - 8.0 / 6.0) < 1e-14


def test_tet_errors():
    rule, _ = reference_element(TET)
    inverted = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, -1]], dtype=float)
    flat = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.5, 0.5, 0]], dtype=float)
    with pytest.raises(InvertedElement):
        jacobian_affine(ElementGeometry(TET, inverted), rule)
    with pytest.raises(DegenerateElement) as err:
        jacobian_affine(ElementGeometry(TET, flat), rule, element_index=7)
    assert err.value.element_index == 7 and err.value.point_index is None
    with pytest.raises(ValueError):
        jacobian_affine(ElementGeometry(PRISM, PRISM.reference_vertices), rule)


def test_prisms():
    rule, table = reference_element(PRISM)
    unit = ElementGeometry(PRISM, PRISM.reference_vertices)
    vols = []
    for q in range(rule.n_points):
        jac = jacobian_at_point(unit, q, rule, table)
        assert abs(jac.det - 1.0) < 1e-14
        vols.append(jac.vol)
    assert abs(sum(vols) - 1.0) < 1e-14
    stretched = PRISM.reference_vertices.copy()
    stretched[:, 2] *= 3.0
    for q in range(rule.n_points):
        assert abs(jacobian_at_point(ElementGeometry(PRISM, stretched), q, rule, table).det - 3.0) < 1e-13
    twisted = PRISM.reference_vertices.copy()
    twisted[4, :2] += (0.2, 0.1)
    dets = [jacobian_at_point(ElementGeometry(PRISM, twisted), q, rule, table).det for q in range(6)]
    assert max(dets) - min(dets) > 1e-3
    flat = PRISM.reference_vertices.copy()
    flat[3:] = flat[:3]
    with pytest.raises(DegenerateElement) as err:
        jacobian_at_point(ElementGeometry(PRISM, flat), 3, rule, table)
    assert err.value.point_index == 3
    with pytest.raises(IndexError):
        jacobian_at_point(unit, 6, rule, table)


def test_random_elements_consistency(rng):
    rule_t, table_t = reference_element(TET)
    rule_p, table_p = reference_element(PRISM)
    for _ in range(10):
        g = random_tet_geometry(rng)
        jac = jacobian_affine(g, rule_t)
        assert np.array_equal(jac.dx_dxi, (g.coords[1:] - g.coords[0]).T)   # the reference's operations
        assert np.abs(jac.dx_dxi @ jac.dxi_dx - np.eye(3)).max() < 1e-12
        assert abs(jac.det - np.linalg.det(jac.dx_dxi)) <= 1e-13 * abs(jac.det)
        gdx = global_derivatives(jac, table_t.local_derivatives[0])
        assert np.abs(gdx.sum(axis=0)).max() < 1e-12
        # generic path on a tet agrees with the affine one
        for q in range(rule_t.n_points):
            jq = jacobian_at_point(g, q, rule_t, table_t)
            assert abs(jq.det - jac.det) <= 1e-14 * abs(jac.det)
        p = random_prism_geometry(rng)
        for q in range(rule_p.n_points):
            jac = jacobian_at_point(p, q, rule_p, table_p)
            assert np.abs(jac.dx_dxi - p.coords.T @ table_p.local_derivatives[q]).max() <= 1e-15 * 8
            assert np.abs(jac.dx_dxi @ jac.dxi_dx - np.eye(3)).max() < 1e-11
