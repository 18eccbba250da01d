"""B200-native element integration for first-order tets and prisms (arXiv 1504.01023).

Drop-in for the hot path of the reference package ``feklab``
(``integrate_batch`` / ``integrate_element``, ``pkg/src/feklab/__init__.py:10-65``):
the same descriptors, batch containers, result type and exceptions, backed by
hand-written sm_100a CUDA kernels in ``libfek.so`` (C-ABI: ``include/fek.h``).
"""

from .errors import (CounterMismatch, DegenerateElement, FeklabError, GeometryError, HeterogeneousBatch,
                     InvertedElement, NativeLibraryError, ShapeMismatch)
from .geometry import DEGENERACY_REL_TOL, ElementGeometry, JacobianData
from .kernels import (BatchResult, DeviceBatch, TrafficCounters, access_breakdown, apply_batch, assemble_batch,
                      csr_pattern, global_accesses, integrate_batch, integrate_element, launch_config,
                      phase_op_counts)
from .layout import (ELEMENT_MAJOR, LANE_WIDTHS, BatchLayout, ElementBatch, LayoutKind, build_batch, convert,
                     extract, flat_length, pack_rows, read_batch, unpack_rows, write_batch)
from .perfmodel import (B200_NOMINAL, BUILTIN_PROFILES, KernelCost, ProcessorProfile, b200_profile, efficiency,
                        kernel_cost, limiting_intensity, memory_requirements, time_bound)
from .problems import (CoefficientSet, ElementMatrix, GeometryPath, KernelDescriptor, ProblemClass, Variant,
                       all_descriptors, case_descriptors, natural_path)
from .refelem import ElementType, QuadratureRule, ShapeFunctionTable, reference_element, shape_at

__version__ = "0.1.0"

__all__ = [
    "B200_NOMINAL", "BUILTIN_PROFILES", "KernelCost", "ProcessorProfile", "b200_profile", "efficiency",
    "kernel_cost", "limiting_intensity", "memory_requirements", "time_bound",
    "BatchLayout", "BatchResult", "apply_batch", "assemble_batch", "csr_pattern", "CoefficientSet", "CounterMismatch", "DEGENERACY_REL_TOL", "DegenerateElement",
    "DeviceBatch", "ELEMENT_MAJOR", "ElementBatch", "ElementGeometry", "JacobianData", "ElementMatrix", "ElementType",
    "FeklabError", "GeometryError", "GeometryPath", "HeterogeneousBatch", "InvertedElement", "KernelDescriptor",
    "LANE_WIDTHS", "LayoutKind", "NativeLibraryError", "ProblemClass", "QuadratureRule", "ShapeFunctionTable",
    "ShapeMismatch", "TrafficCounters", "Variant", "access_breakdown", "all_descriptors", "build_batch",
    "case_descriptors", "convert", "extract", "flat_length", "global_accesses", "integrate_batch",
    "integrate_element", "launch_config", "natural_path", "pack_rows", "phase_op_counts", "read_batch",
    "reference_element", "shape_at", "unpack_rows", "write_batch",
]
