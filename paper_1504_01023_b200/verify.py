"""Correctness gate of the ``verify`` / ``bench`` / ``tune`` commands.

Mirror of ``pkg/src/feklab/verify.py``: a seeded corpus of random
non-degenerate elements, and ``run_verification``, which checks every
requested descriptor's GPU results — ``integrate_element`` on a prefix,
``integrate_batch`` on the whole corpus — against a deliberately naive
per-element integrator within a relative Frobenius tolerance (1e-12).

The corpus generators draw from ``numpy.random.Generator`` in exactly the
reference's order (``verify.py:48-105``), so a seed names the same elements
in both packages.

``integrate_reference`` is the gate's checker: Algorithm 1 of the paper as
the reference states it (``oracle.py:48-92``) — Jacobian and global
derivatives per point, coefficients materialised per point, then the full
(point, row, column, test slot, trial slot) contraction.  It is the one
integrator in this package that runs on the CPU, and it exists only to judge
the CUDA kernels here, as ``feklab.oracle`` does in the reference; no
product entry point (``integrate_batch``, ``integrate_element``) ever calls
it (``tests/test_native_abi.py`` checks that).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DegenerateElement, InvertedElement
from .geometry import DEGENERACY_REL_TOL, ElementGeometry
from .kernels import integrate_batch, integrate_element
from .layout import build_batch
from .problems import CoefficientSet, ElementMatrix, KernelDescriptor, ProblemClass, case_descriptors
from .refelem import ElementType, reference_element

DEFAULT_TOLERANCE = 1e-12


def relative_difference(got, want) -> float:
    """||got - want||_F / ||want||_F; an exact zero reference only matches exact zero (``verify.py:30-40``)."""
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    diff = float(np.linalg.norm(got - want))
    ref = float(np.linalg.norm(want))
    if ref == 0.0:
        return 0.0 if diff == 0.0 else float("inf")
    return diff / ref


def matrices_close(got: ElementMatrix, want: ElementMatrix, tol: float = DEFAULT_TOLERANCE) -> bool:
    return relative_difference(got.A, want.A) <= tol and relative_difference(got.b, want.b) <= tol


# ---------------------------------------------------------------------------
# checker: Algorithm 1 (oracle.py:48-92)
# ---------------------------------------------------------------------------

def _adjugate(m: np.ndarray) -> tuple[np.ndarray, float]:
    """Cofactor adjugate and determinant, ``geometry.py:57-77``'s operation order."""
    (a, b, c), (d, e, f), (g, h, i) = m
    k0, k1, k2 = e * i - f * h, f * g - d * i, d * h - e * g
    adj = np.array([[k0, c * h - b * i, b * f - c * e],
                    [k1, a * i - c * g, c * d - a * f],
                    [k2, b * g - a * h, a * e - b * d]])
    return adj, float(a * k0 + b * k1 + c * k2)


def _point_jacobian_det(coords: np.ndarray, ld_q: np.ndarray) -> tuple[np.ndarray, float]:
    return _adjugate(coords.T @ ld_q)


def _classify(det: float, scale: float, q: int) -> None:
    tol = DEGENERACY_REL_TOL * scale ** 3
    if abs(det) <= tol:
        raise DegenerateElement(f"|det J| = {abs(det):.3e} <= {tol:.3e}", None, q)
    if det < 0.0:
        raise InvertedElement(f"det J = {det:.3e} < 0", None, q)


def materialize_coefficients(coeff: CoefficientSet, n_quad: int) -> tuple[np.ndarray, np.ndarray]:
    """Dense per-point ``c[i][j][q]``, ``d[i][q]`` (``oracle.py:29-45``).

    Poisson: identity diffusion on the derivative slots, ``d0[q]`` in ``d[0]``;
    ConvDiff: the element constants broadcast to every point.
    """
    c = np.zeros((4, 4, n_quad))
    d = np.zeros((4, n_quad))
    if coeff.problem is ProblemClass.POISSON:
        c[1, 1], c[2, 2], c[3, 3] = 1.0, 1.0, 1.0
        d[0] = coeff.d0
    else:
        c[:] = np.asarray(coeff.c)[:, :, None]
        d[:] = np.asarray(coeff.d)[:, None]
    return c, d


def integrate_reference(geom: ElementGeometry, coeff: CoefficientSet) -> ElementMatrix:
    """Naive generic integrator for one element: the gate's checker (never a product path)."""
    etype = geom.element
    rule, table = reference_element(etype)
    nq, ns = etype.n_quad, etype.n_shape
    scale = geom.bounding_box_scale()
    vol = np.empty(nq)
    phi = np.empty((4, ns, nq))          # slot 0: value, slots 1..3: global derivatives
    for q in range(nq):
        adj, det = _point_jacobian_det(geom.coords, table.local_derivatives[q])
        _classify(det, scale, q)
        inv = adj / det
        vol[q] = det * rule.weights[q]
        phi[0, :, q] = table.values[q]
        phi[1:, :, q] = (table.local_derivatives[q] @ inv).T
    c, d = materialize_coefficients(coeff, nq)
    A = np.einsum("q,ijq,irq,jsq->rs", vol, c, phi, phi)
    b = np.einsum("q,iq,irq->r", vol, d, phi)
    return ElementMatrix(A, b)


# ---------------------------------------------------------------------------
# corpus (verify.py:48-105, same draw order)
# ---------------------------------------------------------------------------

def random_tet_geometry(rng: np.random.Generator) -> ElementGeometry:
    """Positively oriented tet, |det(edges)| >= 0.05 (orientation fixed by swapping two edges)."""
    while True:
        v0 = rng.uniform(-1.0, 1.0, size=3)
        edges = rng.uniform(-1.0, 1.0, size=(3, 3))
        det = np.linalg.det(edges)
        if abs(det) < 0.05:
            continue
        if det < 0.0:
            edges[[1, 2]] = edges[[2, 1]]
        return ElementGeometry(ElementType.TETRAHEDRON, np.vstack([v0, v0 + edges]))


def random_prism_geometry(rng: np.random.Generator, twist: float = 0.15) -> ElementGeometry:
    """Affine image of the reference prism plus ``twist``-scaled vertex jitter.

    Redrawn until det J > 1e-3 * diag^3 at every quadrature point (which also
    rules out the degenerate / inverted outcomes the reference catches).
    """
    ref = ElementType.PRISM.reference_vertices
    _, table = reference_element(ElementType.PRISM)
    while True:
        linear = rng.uniform(-1.0, 1.0, size=(3, 3))
        if np.linalg.det(linear) < 0.05:
            continue
        shift = rng.uniform(-1.0, 1.0, size=3)
        coords = ref @ linear.T + shift
        coords = coords + twist * rng.uniform(-1.0, 1.0, size=coords.shape)
        geom = ElementGeometry(ElementType.PRISM, coords)
        dets = [_point_jacobian_det(geom.coords, ld)[1] for ld in table.local_derivatives]
        if min(dets) > 1e-3 * geom.bounding_box_scale() ** 3:
            return geom


def random_geometry(etype: ElementType, rng: np.random.Generator) -> ElementGeometry:
    return random_tet_geometry(rng) if etype is ElementType.TETRAHEDRON else random_prism_geometry(rng)


def random_coefficients(problem: ProblemClass, etype: ElementType, rng: np.random.Generator) -> CoefficientSet:
    return CoefficientSet.from_flat(problem, etype, rng.uniform(-1.0, 1.0, size=problem.coefficient_size(etype)))


# ---------------------------------------------------------------------------
# reports
# ---------------------------------------------------------------------------

@dataclass
class CaseReport:
    element: ElementType
    problem: ProblemClass
    n_elements: int
    max_rel_err: float
    failures: list[str] = field(default_factory=list)

    @property
    def passed(self) -> bool:
        return not self.failures


@dataclass
class VerificationReport:
    tolerance: float
    cases: list[CaseReport] = field(default_factory=list)

    @property
    def passed(self) -> bool:
        return all(c.passed for c in self.cases)

    @property
    def max_rel_err(self) -> float:
        return max((c.max_rel_err for c in self.cases), default=0.0)

    def summary_lines(self) -> list[str]:
        out = []
        for c in self.cases:
            out.append(f"{c.element.value}/{c.problem.value}: {'ok' if c.passed else 'FAIL'} "
                       f"({c.n_elements} elements, max rel err {c.max_rel_err:.2e})")
            out.extend(f"  {msg}" for msg in c.failures[:5])
        return out


def _element_error(got: ElementMatrix, want: ElementMatrix) -> float:
    return max(relative_difference(got.A, want.A), relative_difference(got.b, want.b))


def run_verification(per_case: int = 200, seed: int = 20240301, tolerance: float = DEFAULT_TOLERANCE,
                     descriptors: list[KernelDescriptor] | None = None) -> VerificationReport:
    """Check GPU results of ``descriptors`` (default: all 18) against the checker (``verify.py:150-216``).

    Cases run in (element, problem) name order from one generator, so the
    corpus of each case matches the reference's for the same seed.  Per
    descriptor: ``integrate_element`` on the first min(per_case, 16)
    elements (one device launch each) and ``integrate_batch`` on the whole
    corpus (one launch).
    """
    report = VerificationReport(tolerance=tolerance)
    cases: dict = {}
    for desc in descriptors or ():
        cases.setdefault((desc.element, desc.problem), []).append(desc)
    if not cases:
        cases = {(e, p): list(case_descriptors(e, p)) for e in ElementType for p in ProblemClass}
    rng = np.random.default_rng(seed)
    for (element, problem), descs in sorted(cases.items(), key=lambda kv: (kv[0][0].value, kv[0][1].value)):
        corpus = [(random_geometry(element, rng), random_coefficients(problem, element, rng))
                  for _ in range(per_case)]
        want = [integrate_reference(g, c) for g, c in corpus]
        case = CaseReport(element, problem, per_case, 0.0)
        batch = build_batch(corpus)
        for desc in descs:
            for i in range(min(per_case, 16)):
                err = _element_error(integrate_element(desc, *corpus[i]), want[i])
                case.max_rel_err = max(case.max_rel_err, err)
                if err > tolerance:
                    case.failures.append(f"{desc.short_name()} element {i}: rel err {err:.2e}")
            result = integrate_batch(desc, batch)
            for i in range(per_case):
                err = _element_error(result.element_matrix(i), want[i])
                case.max_rel_err = max(case.max_rel_err, err)
                if err > tolerance:
                    case.failures.append(f"{desc.short_name()} batch element {i}: rel err {err:.2e}")
        report.cases.append(case)
    return report
