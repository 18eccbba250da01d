"""Cost-model constants: algorithmic traffic and flops per element.

Mirror of ``pkg/src/feklab/kernels/counts.py:40-114`` (Table 4 of the paper,
``PAPER.md:735-756``).  These are the roofline numerators of ``bench.py``:

* bytes/element = ``global_accesses * sizeof(real)`` — geometry and
  coefficients read once, stiffness and load written once (36/66/52/80
  reals for tet/P, prism/P, tet/CD, prism/CD);
* flops/element = the QSS model total (290/2700/986/4806), used for every
  variant so wasteful loop orders do not earn a higher ceiling.
"""

from __future__ import annotations

from dataclasses import dataclass

from ..problems import KernelDescriptor, ProblemClass, Variant
from ..refelem import ElementType

_T, _P = ElementType.TETRAHEDRON, ElementType.PRISM
_PO, _CD = ProblemClass.POISSON, ProblemClass.CONV_DIFF

# (tet/P, prism/P, tet/CD, prism/CD) per variant — Table 4, counts.py:40-53
_TABLE4 = {
    Variant.QSS: (290, 2700, 986, 4806),
    Variant.SQS: (290, 10416, 986, 12492),
    Variant.SSQ: (290, 54876, 1623, 65232),
}
OP_TOTALS: dict[tuple[Variant, ElementType, ProblemClass], int] = {
    (v, e, p): row[i]
    for v, row in _TABLE4.items()
    for i, (e, p) in enumerate(((_T, _PO), (_P, _PO), (_T, _CD), (_P, _CD)))
}

GEO_DERIV_OPS = {_T: 9, _P: 126}
JACOBIAN_OPS = 49
SHAPE_DERIV_OPS = {_T: 60, _P: 90}
SHAPE_DERIV_OPS_PER_FN = 15


def access_breakdown(element: ElementType, problem: ProblemClass) -> tuple[int, int, int, int]:
    """(geometry reads, coefficient reads, stiffness writes, load writes) in reals."""
    ns = element.n_shape
    return element.geometry_size, problem.coefficient_size(element), ns * ns, ns


def global_accesses(element: ElementType, problem: ProblemClass) -> int:
    return sum(access_breakdown(element, problem))


@dataclass(frozen=True)
class PhaseOpCounts:
    geo_derivs: int
    jacobian_terms: int
    shape_derivs: int
    final_update: int
    total: int


def phase_op_counts(desc: KernelDescriptor) -> PhaseOpCounts:
    """Per-phase split of the model total (counts.py:88-114)."""
    total = OP_TOTALS[(desc.variant, desc.element, desc.problem)]
    if desc.element is _T:
        geo, jac, shape = GEO_DERIV_OPS[_T], JACOBIAN_OPS, SHAPE_DERIV_OPS[_T]
    else:
        nq, ns = desc.element.n_quad, desc.element.n_shape
        reps = {Variant.QSS: nq, Variant.SQS: ns * nq, Variant.SSQ: ns * ns * nq}[desc.variant]
        if desc.variant is Variant.SSQ:
            shape = 2 * SHAPE_DERIV_OPS_PER_FN * reps
        else:
            shape = SHAPE_DERIV_OPS[_P] * reps
        geo, jac = GEO_DERIV_OPS[_P] * reps, JACOBIAN_OPS * reps
    return PhaseOpCounts(geo, jac, shape, total - geo - jac - shape, total)


def algorithmic_bytes(element: ElementType, problem: ProblemClass, real_bytes: int = 8) -> int:
    return global_accesses(element, problem) * real_bytes


def algorithmic_flops(element: ElementType, problem: ProblemClass) -> int:
    return OP_TOTALS[(Variant.QSS, element, problem)]
