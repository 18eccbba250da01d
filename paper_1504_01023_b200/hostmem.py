"""Host staging memory: page-locked numpy arrays for the H2D/D2H pipeline.

Large host buffers that cross the PCIe link (batch inputs built by this
package, result arrays returned by ``integrate_batch``) are allocated
page-locked through torch's caching host allocator, so the copy engines can
DMA them asynchronously and repeated calls reuse the same pinned blocks
instead of paying ``cudaHostAlloc`` every time.  Small arrays, and every array
on a machine without a CUDA driver, are ordinary numpy memory.
"""

from __future__ import annotations

import numpy as np

PIN_THRESHOLD_BYTES = 1 << 22  # 4 MiB

_pin_ok: bool | None = None


def _pinning_available() -> bool:
    global _pin_ok
    if _pin_ok is None:
        try:
            import torch

            _pin_ok = bool(torch.cuda.is_available())
        except Exception:  # pragma: no cover - torch is a hard dependency
            _pin_ok = False
    return _pin_ok


def empty(shape, dtype=np.float64, pin: bool | None = None) -> np.ndarray:
    """Uninitialised host array; page-locked when large and CUDA is present."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    if pin is None:
        pin = count * dtype.itemsize >= PIN_THRESHOLD_BYTES
    if pin and _pinning_available():
        import torch

        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}[dtype]
        t = torch.empty(count, dtype=tdt, pin_memory=True)
        return t.numpy().reshape(shape)
    return np.empty(shape, dtype=dtype)


def is_pinned(arr: np.ndarray) -> bool:
    """True when ``arr``'s memory is page-locked (as seen by the CUDA runtime)."""
    if not _pinning_available():
        return False
    import torch

    try:
        return bool(torch.from_numpy(np.asarray(arr)).is_pinned())
    except Exception:
        return False
