"""Element geometry container and the degeneracy tolerance.

Mirror of the parts of ``pkg/src/feklab/geometry.py`` that sit on the API of
the hot path: ``ElementGeometry`` (``geometry.py:27-46``, the argument type of
``integrate_element``) and ``DEGENERACY_REL_TOL`` (``geometry.py:22-24``),
which the CUDA kernels apply as ``|det J| <= 1e-14 * diag**3`` with ``diag``
the bounding-box diagonal (``batched.py:136-148,166-177``).

The scalar Jacobian routines of the reference are not mirrored here: the
product computes Jacobians on the device only; the CPU restatement used to
check it lives in ``oracle/``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .refelem import ElementType

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
