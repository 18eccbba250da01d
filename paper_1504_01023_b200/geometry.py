"""Element geometry: container, degeneracy tolerance, and per-element Jacobians.

Mirror of ``pkg/src/feklab/geometry.py``:

* ``ElementGeometry`` (``geometry.py:27-46``, the argument type of
  ``integrate_element``);
* ``DEGENERACY_REL_TOL`` (``geometry.py:22-24``), which the CUDA kernels
  apply as ``|det J| <= 1e-14 * diag**3`` with ``diag`` the bounding-box
  diagonal (``batched.py:136-148,166-177``);
* ``JacobianData``, ``jacobian_affine`` and ``jacobian_at_point``
  (``geometry.py:49-138``).  The Jacobian, its inverse and det J are
  computed on the GPU by ``fek_jacobian`` (one thread, the kernels' own
  reference-exact Jacobian arithmetic); only ``vol = det * w`` is formed
  here.  Errors are raised as the reference does: degenerate first, then
  inverted, carrying the element and point index.
* ``global_derivatives`` (``geometry.py:141-143``): the chain rule on an
  already-computed ``JacobianData``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import errors as _errors
from .refelem import ElementType, QuadratureRule, ShapeFunctionTable

DEGENERACY_REL_TOL = 1e-14


@dataclass(frozen=True)
class ElementGeometry:
    element: ElementType
    coords: np.ndarray  # (n_vertices, 3)

    def __post_init__(self):
        arr = np.ascontiguousarray(self.coords, dtype=np.float64)
        want = (self.element.n_vertices, 3)
        if arr.shape != want:
            raise ValueError(f"{self.element.value} geometry must have shape {want}, got {arr.shape}")
        object.__setattr__(self, "coords", arr)

    def bounding_box_scale(self) -> float:
        span = self.coords.max(axis=0) - self.coords.min(axis=0)
        return float(np.sqrt(np.dot(span, span)))


@dataclass(frozen=True)
class JacobianData:
    """Jacobian terms of the reference-to-real mapping (``geometry.py:49-64``).

    ``vol`` is det J times the quadrature weight(s): a per-point array on the
    affine path and a scalar on the point-local path.
    """

    dx_dxi: np.ndarray  # (3, 3): dx_i / dxi_k
    dxi_dx: np.ndarray  # (3, 3): dxi_k / dx_i
    det: float
    vol: np.ndarray | float


def _device_jacobian(geom: ElementGeometry, point: int) -> tuple[np.ndarray, np.ndarray, float, float]:
    import torch

    from . import _native
    from .problems import GeometryPath, KernelDescriptor, ProblemClass, Variant
    from .kernels.batched import _desc_struct
    from .layout import ELEMENT_MAJOR

    lib = _native.load()
    et = geom.element
    g = torch.tensor(np.asarray(geom.coords, dtype=np.float64).reshape(-1), device="cuda")
    out = torch.empty(20, dtype=torch.float64, device=g.device)
    path = GeometryPath.GEO_LINEAR if point < 0 else GeometryPath.GEO_GENERIC
    desc = KernelDescriptor(Variant.QSS, path, ProblemClass.POISSON, et)
    dd = _desc_struct(desc, ELEMENT_MAJOR, 1, 0, _native.DTYPE["float64"], g.data_ptr(), 0, 0, 0, 0)
    stream = torch.cuda.current_stream()
    _native.check(lib.fek_jacobian(ctypes.byref(dd), 0, point, out.data_ptr(), stream.cuda_stream), "fek_jacobian")
    host = out.cpu().numpy()
    return host[:9].reshape(3, 3).copy(), host[9:18].reshape(3, 3).copy(), float(host[18]), float(host[19])


def _check(det: float, tol: float, element_index, point_index) -> None:
    """Degenerate first, then inverted (``geometry.py:81-91``)."""
    if abs(det) <= tol:
        raise _errors.DegenerateElement(f"|det J| = {abs(det):.3e} <= {tol:.3e}", element_index, point_index)
    if det < 0.0:
        raise _errors.InvertedElement(f"det J = {det:.3e} < 0", element_index, point_index)


def jacobian_affine(geom: ElementGeometry, rule: QuadratureRule, element_index=None) -> JacobianData:
    """Constant Jacobian of an affine tetrahedron; ``vol`` = det J * w per point (``geometry.py:94-112``)."""
    if geom.element is not ElementType.TETRAHEDRON:
        raise ValueError("affine path only applies to tetrahedra")
    J, inv, det, tol = _device_jacobian(geom, -1)
    _check(det, tol, element_index, None)
    return JacobianData(J, inv, det, det * np.asarray(rule.weights))


def jacobian_at_point(geom: ElementGeometry, q: int, rule: QuadratureRule, table: ShapeFunctionTable,
                      element_index=None) -> JacobianData:
    """Jacobian at quadrature point ``q``; errors carry the point (``geometry.py:115-138``)."""
    if not 0 <= q < rule.n_points:
        raise IndexError(f"quadrature point {q} out of range")
    J, inv, det, tol = _device_jacobian(geom, q)
    _check(det, tol, element_index, q)
    return JacobianData(J, inv, det, float(det * rule.weights[q]))


def global_derivatives(jac: JacobianData, local_derivs: np.ndarray) -> np.ndarray:
    """Chain rule d phi_s / d x_i = sum_k local[s, k] dxi_dx[k, i] (``geometry.py:141-143``)."""
    return np.asarray(local_derivs) @ jac.dxi_dx
