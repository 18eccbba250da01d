"""Exception types raised across the drop-in boundary.

Mirrors the reference hierarchy (``pkg/src/feklab/errors.py:4-39``) name for
name so callers that catch ``feklab`` exceptions keep working after the switch:

* ``GeometryError(message, element_index, point_index)`` renders its message
  as ``"<message> @ element <i> @ quadrature point <q>"`` (``errors.py:8-19``);
* ``DegenerateElement`` / ``InvertedElement`` are raised by the device kernels'
  error word (decoded on the host, see ``kernels/batched.py``);
* ``ShapeMismatch``, ``HeterogeneousBatch``, ``CounterMismatch`` as in the
  reference.

``NativeLibraryError`` is new: the CUDA library is missing, failed to load, or
returned a launch error.  There is no CPU fallback, so this is raised loudly.
"""

from __future__ import annotations


class FeklabError(Exception):
    """Root of every error this package raises on purpose."""


class GeometryError(FeklabError):
    """Invalid element geometry, located by element and quadrature point."""

    def __init__(self, message, element_index=None, point_index=None):
        self.element_index = element_index
        self.point_index = point_index
        text = str(message)
        if element_index is not None:
            text += f" @ element {element_index}"
        if point_index is not None:
            text += f" @ quadrature point {point_index}"
        super().__init__(text)


class DegenerateElement(GeometryError):
    """|det J| is at or below the scale-relative tolerance."""


class InvertedElement(GeometryError):
    """det J < 0: the element is mapped with flipped orientation."""


class ShapeMismatch(FeklabError):
    """Batch or element data disagrees with the kernel descriptor."""


class HeterogeneousBatch(FeklabError):
    """A batch was assembled from elements of different type or problem."""


class CounterMismatch(FeklabError):
    """Traffic counters disagree with the 36/66/52/80 cost model."""


class NativeLibraryError(FeklabError, RuntimeError):
    """libfek.so is unavailable or a CUDA call behind the C-ABI failed."""


BOUNDARY_TYPES = ("GeometryError", "DegenerateElement", "InvertedElement", "ShapeMismatch")


def bind_exception_types(namespace) -> None:
    """Raise a host package's own exception classes across the boundary.

    ``integrate_batch`` / ``integrate_element`` / the geometry helpers look the
    classes up here at raise time, so after ``bind_exception_types(feklab.errors)``
    a feklab caller catching ``feklab.errors.DegenerateElement`` catches the
    drop-in's errors unchanged.  The classes must take
    ``(message, element_index, point_index)`` as the reference's do (``errors.py:8-19``).
    """
    g = globals()
    for name in BOUNDARY_TYPES:
        g[name] = getattr(namespace, name)
