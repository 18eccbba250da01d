"""Per-element API: ``integrate_element`` on the GPU.

Mirror of ``pkg/src/feklab/kernels/scalar.py:242-264``: same descriptor and
shape checks (``ShapeMismatch``), same geometry errors.  The element is run
as a one-element batch through the same CUDA kernel as ``integrate_batch``,
so a batch of identical elements is bitwise equal to ``integrate_element``
(``test_kernels.py:240-248``).  There is no CPU path.
"""

from __future__ import annotations

from .. import errors as _errors
from ..layout import build_batch
from ..problems import ElementMatrix, ProblemClass, coerce_descriptor, coerce_element, coerce_problem
from .batched import integrate_batch


def integrate_element(desc, geom, coeff) -> ElementMatrix:
    desc = coerce_descriptor(desc)
    if coerce_element(geom.element) is not desc.element:
        raise _errors.ShapeMismatch(f"descriptor expects {desc.element.value}, geometry is {geom.element.value}")
    if coerce_problem(coeff.problem) is not desc.problem:
        raise _errors.ShapeMismatch(f"descriptor expects {desc.problem.value}, coefficients are {coeff.problem.value}")
    if desc.problem is ProblemClass.POISSON and len(coeff.d0) != desc.element.n_quad:
        raise _errors.ShapeMismatch(f"expected {desc.element.n_quad} right-hand-side values, got {len(coeff.d0)}")
    return integrate_batch(desc, build_batch([(geom, coeff)])).element_matrix(0)
