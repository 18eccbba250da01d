"""ctypes binding of libfek.so (the C-ABI declared in include/fek.h).

There is no CPU fallback: if the library is missing or cannot be loaded,
every entry point raises ``NativeLibraryError``.  ``load()`` is also how the
tests prove the in-tree ``.so`` (not something in site-packages) is the code
that runs.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeLibraryError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfek.so")
if os.environ.get("FEK_LIB_OVERRIDE"):  # kernel-tuning experiments only
    LIB_PATH = os.path.abspath(os.environ["FEK_LIB_OVERRIDE"])
HEADER_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fek.h")

ABI_VERSION = 4
NO_ERROR = 0xFFFFFFFFFFFFFFFF

OK, ERR_ARGUMENT, ERR_ALIGNMENT, ERR_CUDA, ERR_WORKSPACE, ERR_GEOMETRY = range(6)
KIND_DEGENERATE, KIND_INVERTED, KIND_PIPELINE_TIMEOUT, KIND_NEAR, KIND_PATTERN = 1, 2, 3, 4, 5

# enum codes (fek.h)
ELEMENT = {"tet": 0, "prism": 1}
PROBLEM = {"poisson": 0, "convdiff": 1}
VARIANT = {"qss": 0, "sqs": 1, "ssq": 2}
GEO_PATH = {"linear": 0, "generic": 1}
DTYPE = {"float64": 0, "float32": 1}
LAYOUT = {"major": 0, "interleaved": 1}
OUT_SPLIT, OUT_PACKED = 0, 1


class BatchDesc(ctypes.Structure):
    _fields_ = [
        ("element", ctypes.c_int32),
        ("problem", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("geometry_path", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("layout", ctypes.c_int32),
        ("lane_width", ctypes.c_int32),
        ("out_format", ctypes.c_int32),
        ("n_elements", ctypes.c_int64),
        ("base_index", ctypes.c_int64),
        ("geometry", ctypes.c_void_p),
        ("coefficients", ctypes.c_void_p),
        ("stiffness", ctypes.c_void_p),
        ("load", ctypes.c_void_p),
        ("error_key", ctypes.c_void_p),
        ("out_lane_width", ctypes.c_int32),
        ("ctas_per_sm", ctypes.c_int32),
        ("scheduler", ctypes.c_void_p),
        ("tile_elements", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


# name -> (restype, argtypes); must cover every function fek.h declares
_P = ctypes.c_void_p
_DP = ctypes.POINTER(BatchDesc)
SIGNATURES = {
    "fek_abi_version": (ctypes.c_int, []),
    "fek_batch_desc_size": (ctypes.c_size_t, []),
    "fek_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "fek_last_cuda_error": (ctypes.c_char_p, []),
    "fek_integrate": (ctypes.c_int, [_DP, _P]),
    "fek_launch_config": (ctypes.c_int, [_DP, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "fek_host_workspace_bytes": (ctypes.c_size_t, [_DP, ctypes.c_int, ctypes.c_int64]),
    "fek_integrate_host": (ctypes.c_int, [_DP, _P, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_P),
                                          ctypes.c_int64, ctypes.POINTER(ctypes.c_ulonglong)]),
    "fek_host_staging_bytes": (ctypes.c_size_t, [_DP, ctypes.c_int, ctypes.c_int64]),
    "fek_integrate_host_staged": (ctypes.c_int, [_DP, _P, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_P),
                                                 ctypes.c_int64, _P, ctypes.c_size_t, ctypes.c_int,
                                                 ctypes.POINTER(ctypes.c_ulonglong)]),
    "fek_decode_error": (ctypes.c_int, [ctypes.c_ulonglong, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
    "fek_classify": (ctypes.c_int, [_DP, _P]),
    "fek_apply": (ctypes.c_int, [_DP, _P, _P, _P, _P, _P]),
    "fek_assemble": (ctypes.c_int, [_DP, _P, _P, _P, _P, _P, _P]),
    "fek_error_detail": (ctypes.c_int, [_DP, ctypes.c_int64, ctypes.c_int32, _P, _P]),
    "fek_jacobian": (ctypes.c_int, [_DP, ctypes.c_int64, ctypes.c_int32, _P, _P]),
    "fek_checksum_scratch_bytes": (ctypes.c_size_t, []),
    "fek_checksum": (ctypes.c_int, [_DP, _P, _P, _P, _P]),
    "fek_pcg64_uniform": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_double, ctypes.c_double, _P, _P]),
    "fek_mesh_geometry": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_ulonglong),
                                         ctypes.c_double, _P, _P]),
    "fek_convert_layout": (ctypes.c_int, [_P, ctypes.c_int32, _P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_double, _P]),
}

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load (once) and type the in-tree libfek.so; raise if it is unusable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -m paper_1504_01023_b200.build_native` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        if lib.fek_abi_version() != ABI_VERSION:
            raise NativeLibraryError(f"libfek ABI {lib.fek_abi_version()} != expected {ABI_VERSION}")
        if lib.fek_batch_desc_size() != ctypes.sizeof(BatchDesc):
            raise NativeLibraryError(f"fek_batch_desc is {lib.fek_batch_desc_size()} bytes in libfek, "
                                     f"{ctypes.sizeof(BatchDesc)} in the ctypes binding")
        _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status == OK:
        return
    lib = load()
    msg = lib.fek_status_string(status).decode()
    if status == ERR_CUDA:
        msg += f" ({lib.fek_last_cuda_error().decode()})"
    raise NativeLibraryError(f"{what}: {msg}")


def decode_error(key: int) -> tuple[int, int | None, int]:
    """(element, point or None, kind) of an error word."""
    lib = load()
    e, q, k = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
    check(lib.fek_decode_error(ctypes.c_ulonglong(key), ctypes.byref(e), ctypes.byref(q), ctypes.byref(k)),
          "fek_decode_error")
    return e.value, (None if q.value < 0 else q.value), k.value


def header_functions() -> list[str]:
    """Names of the functions include/fek.h declares (for the export test)."""
    import re

    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_ ]+\**\s*\**(fek_[a-z0-9_]+)\s*\(", text, re.M)))
