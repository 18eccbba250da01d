"""Batch integration drop-in: ``integrate_batch`` on B200 through libfek.so.

Mirror of ``pkg/src/feklab/kernels/batched.py:53-106,536-606``.  Same call,
same result type, same errors:

    integrate_batch(desc, batch, out_layout=ELEMENT_MAJOR, workers=1) -> BatchResult

* ``batch`` may be a host ``ElementBatch`` (ours, or the reference's own —
  fields are duck-typed) or a ``DeviceBatch`` whose flat arrays are CUDA
  tensors.  Host batches stream through ``fek_integrate_host`` (chunked
  H2D -> kernel -> D2H on three CUDA streams) and come back as numpy arrays,
  so a reference caller sees no difference; device batches stay on the GPU
  (``fek_integrate`` on the current torch stream) and return torch tensors.
* ``workers`` does not change the launch (the GPU decides the parallel
  decomposition; results are bitwise independent of it, as the reference
  promises for its thread count, ``batched.py:10-13``).  It does change which
  error is reported, exactly as in the reference: with ``workers > 1`` the batch
  is split ``np.linspace(0, n, workers+1)``, each range applies the first-error
  rule with 8192-element blocks counted from its own start, and the error with
  the smallest element index wins (``batched.py:569-599``).  The GPU replays
  that on the (rare) error path with one exact classification pass per range.
* A degenerate/inverted element raises ``DegenerateElement`` /
  ``InvertedElement`` with the reference's element/point indices and message
  text; there is no partial result (``batched.py:544-547``).
* There is no CPU fallback: without the CUDA library or a GPU this raises
  ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from .. import _native, hostmem
from .. import errors as _errors
from ..errors import NativeLibraryError
from ..layout import (ELEMENT_MAJOR, BatchLayout, ElementBatch, LayoutKind, coerce_layout, flat_length, pack_rows,
                      unpack_rows)
from ..problems import (ElementMatrix, KernelDescriptor, ProblemClass, coerce_descriptor, coerce_element,
                        coerce_problem)
from ..refelem import ElementType

HOST_STREAMS = 3


@dataclass
class TrafficCounters:
    """Reals moved per batch (``batched.py:53-80``): inputs read once, outputs written once."""

    geometry_reads: int = 0
    coefficient_reads: int = 0
    stiffness_writes: int = 0
    load_writes: int = 0

    @property
    def total(self) -> int:
        return self.geometry_reads + self.coefficient_reads + self.stiffness_writes + self.load_writes

    def per_element(self, n_elements: int) -> float:
        return self.total / n_elements

    def breakdown_per_element(self, n_elements: int) -> tuple[float, float, float, float]:
        return (self.geometry_reads / n_elements, self.coefficient_reads / n_elements,
                self.stiffness_writes / n_elements, self.load_writes / n_elements)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class BatchResult:
    """Stiffness matrices (n, ns, ns) and load vectors (n, ns) of a batch.

    numpy arrays for host batches, CUDA tensors for device batches.
    """

    descriptor: KernelDescriptor
    n_elements: int
    stiffness: object
    load: object
    traffic: TrafficCounters
    out_layout: BatchLayout = field(default=ELEMENT_MAJOR)
    # packed rows [A | b] in out_layout, written by the kernel (integrate_batch(..., packed=True));
    # stiffness/load are then zero-copy views (element-major) or None (interleaved)
    flat: object = None

    def _materialize(self) -> None:
        """Unpack stiffness/load from kernel-packed interleaved rows on first use."""
        if self.stiffness is not None or self.flat is None:
            return
        ns = self.descriptor.element.n_shape
        ds, n = ns * ns + ns, self.n_elements
        layout = coerce_layout(self.out_layout)
        if _is_torch(self.flat):
            w = layout.lane_width
            rows = self.flat.view(-1, ds, w).transpose(1, 2).reshape(-1, ds)[:n].contiguous()
        else:
            from ..layout import unpack_rows

            rows = unpack_rows(self.flat, n, ds, layout)
        self.stiffness = rows[:, : ns * ns].reshape(n, ns, ns)
        self.load = rows[:, ns * ns:]

    def check_errors(self) -> None:
        """For a device result made with ``check=False`` (e.g. inside a CUDA graph): read the
        error word (synchronises), resolve a NEAR key with the exact pass, and raise the
        reference's exception if an element is degenerate or inverted."""
        launch = getattr(self, "_launch", None)
        if launch is None:
            return
        import torch

        dd, _, base_index = launch
        stream = torch.cuda.current_stream().cuda_stream  # where the caller ran / replayed the launch
        key = resolve_error_key(dd, self.error_word, stream)
        if key != _native.NO_ERROR:
            _raise_geometry(key, lambda e, q: _device_error_detail(dd, e - base_index, q, stream))

    def element_matrix(self, e: int) -> ElementMatrix:
        if not 0 <= e < self.n_elements:
            raise IndexError(f"element index {e} out of range")
        self._materialize()
        A, b = self.stiffness[e], self.load[e]
        if _is_torch(A):
            A, b = A.detach().cpu().numpy(), b.detach().cpu().numpy()
        return ElementMatrix(np.array(A, dtype=np.float64), np.array(b, dtype=np.float64))

    def output_rows(self):
        """(n, ns*ns + ns) rows: stiffness entries then load (``batched.py:99-102``)."""
        self._materialize()
        n = self.n_elements
        if _is_torch(self.stiffness):
            import torch

            return torch.cat([self.stiffness.reshape(n, -1), self.load], dim=1)
        return np.concatenate([np.asarray(self.stiffness).reshape(n, -1), np.asarray(self.load)], axis=1)

    def flat_output(self, pad_value: float = np.nan):
        """Rows flattened in ``out_layout`` (``batched.py:104-106``); stays on the device for device results.

        For kernel-packed results (``packed=True``) this is the kernel's own
        output buffer (no repacking pass); pad lanes hold NaN unless another
        ``pad_value`` is requested.
        """
        layout = coerce_layout(self.out_layout)
        if self.flat is not None:
            if layout.kind is LayoutKind.ELEMENT_MAJOR or self.n_elements % layout.lane_width == 0 \
                    or np.isnan(pad_value):
                return self.flat
            out = self.flat.clone() if _is_torch(self.flat) else self.flat.copy()
            ds = self.descriptor.element.n_shape * (self.descriptor.element.n_shape + 1)
            w, n = layout.lane_width, self.n_elements
            blk = out.reshape(-1, ds, w)
            blk[-1, :, n % w:] = pad_value
            return out
        rows = self.output_rows()
        if not _is_torch(rows):
            return pack_rows(rows, layout, pad_value)
        import torch

        n, ds = rows.shape
        if layout.kind is LayoutKind.ELEMENT_MAJOR:
            return rows.reshape(-1).clone()
        w = layout.lane_width
        out = torch.full((flat_length(n, ds, layout),), pad_value, dtype=rows.dtype, device=rows.device)
        blocks = -(-n // w)
        padded = torch.full((blocks * w, ds), pad_value, dtype=rows.dtype, device=rows.device)
        padded[:n] = rows
        out.copy_(padded.reshape(blocks, w, ds).transpose(1, 2).reshape(-1))
        return out

    def to_host(self) -> "BatchResult":
        self._materialize()
        if not _is_torch(self.stiffness):
            return self
        return BatchResult(self.descriptor, self.n_elements, self.stiffness.cpu().numpy(),
                           self.load.cpu().numpy(), self.traffic, self.out_layout)


@dataclass(frozen=True)
class DeviceBatch:
    """A batch whose flat geometry/coefficient arrays are CUDA tensors (fp64 or fp32).

    Same storage schemes as ``ElementBatch`` (``layout.py:1-23``).
    """

    element_type: ElementType
    problem: ProblemClass
    n_elements: int
    layout: BatchLayout
    geometry_data: object   # torch.Tensor, flat
    coefficient_data: object

    def __post_init__(self):
        import torch

        for name, t, ds in (("geometry_data", self.geometry_data, self.element_type.geometry_size),
                            ("coefficient_data", self.coefficient_data,
                             self.problem.coefficient_size(self.element_type))):
            if not isinstance(t, torch.Tensor) or not t.is_cuda:
                raise TypeError(f"{name} must be a CUDA tensor")
            want = flat_length(self.n_elements, ds, self.layout)
            if tuple(t.shape) != (want,) or not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous and flat with {want} entries, got {tuple(t.shape)}")
            if t.dtype not in (torch.float64, torch.float32):
                raise TypeError(f"{name} must be float64 or float32")
        if self.geometry_data.dtype != self.coefficient_data.dtype:
            raise TypeError("geometry and coefficient dtypes differ")

    @property
    def dtype(self):
        return self.geometry_data.dtype

    @classmethod
    def from_host(cls, batch, device=None, dtype=None, non_blocking: bool = False) -> "DeviceBatch":
        """Upload a host ``ElementBatch`` (optionally converting to float32)."""
        import torch

        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dtype = dtype or torch.float64

        def up(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            return t.to(device=device, dtype=dtype, non_blocking=non_blocking)

        return cls(coerce_element(batch.element_type), coerce_problem(batch.problem), int(batch.n_elements),
                   coerce_layout(batch.layout), up(batch.geometry_data), up(batch.coefficient_data))

    def convert(self, to: BatchLayout, pad_value: float = np.nan) -> "DeviceBatch":
        """On-device ``layout.convert`` (``layout.py:198-218``): a new batch in layout ``to``.

        The same layout returns copies, as the reference does; otherwise both
        arrays are repacked by ``fek_convert_layout`` with ``pad_value`` in the
        pad lanes of a partial interleaved block.
        """
        import torch

        to = coerce_layout(to)
        if to == self.layout:
            return DeviceBatch(self.element_type, self.problem, self.n_elements, self.layout,
                               self.geometry_data.clone(), self.coefficient_data.clone())
        lib = _native.load()
        dtype = _native.DTYPE["float64" if self.dtype == torch.float64 else "float32"]
        w_in, w_out = self.layout.block, to.block
        out = []
        with torch.cuda.device(self.geometry_data.device):
            stream = torch.cuda.current_stream().cuda_stream
            for src, ds in ((self.geometry_data, self.element_type.geometry_size),
                            (self.coefficient_data, self.problem.coefficient_size(self.element_type))):
                dst = torch.empty(flat_length(self.n_elements, ds, to), dtype=src.dtype, device=src.device)
                _native.check(lib.fek_convert_layout(src.data_ptr(), w_in, dst.data_ptr(), w_out, self.n_elements,
                                                     ds, dtype, float(pad_value), stream), "fek_convert_layout")
                out.append(dst)
        return DeviceBatch(self.element_type, self.problem, self.n_elements, to, *out)

    def to_host(self) -> ElementBatch:
        """Download as a float64 host ``ElementBatch`` in the same layout."""
        import torch

        geo = self.geometry_data.to(torch.float64).cpu().numpy()
        cof = self.coefficient_data.to(torch.float64).cpu().numpy()
        return ElementBatch(self.element_type, self.problem, self.n_elements, self.layout, geo, cof)


def _read_device_batch(path, device, dtype=None, chunk_bytes: int = 64 << 20) -> DeviceBatch:
    """FEKB file -> DeviceBatch through two alternating page-locked staging buffers."""
    import torch

    from ..layout import _read_header

    fh = open(path, "rb")  # an unreadable file fails as OSError before any CUDA call, as on the host path
    try:
        device = torch.device(device)
        if device.index is None:
            device = torch.device(device.type, torch.cuda.current_device())
    except BaseException:
        fh.close()
        raise
    dtype = dtype or torch.float64
    chunk = max(1, chunk_bytes // 8)
    with fh, torch.cuda.device(device):
        etype, problem, layout, n = _read_header(fh, path)
        stream = torch.cuda.Stream(device)
        staging = [torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        scratch = torch.empty(chunk, dtype=torch.float64, device=device) if dtype != torch.float64 else None
        done = [None, None]
        out = []
        k = 0
        for ds in (etype.geometry_size, problem.coefficient_size(etype)):
            size = flat_length(n, ds, layout)
            dst = torch.empty(size, dtype=dtype, device=device)
            for lo in range(0, size, chunk):
                cnt = min(chunk, size - lo)
                slot = k % 2
                if done[slot] is not None:
                    done[slot].synchronize()  # the upload that last used this buffer has finished
                buf = staging[slot][:cnt]
                got = fh.readinto(memoryview(buf.numpy()).cast("B"))
                if got != cnt * 8:
                    raise ValueError(f"{path}: truncated data section")
                with torch.cuda.stream(stream):
                    if scratch is None:
                        dst[lo:lo + cnt].copy_(buf, non_blocking=True)
                    else:
                        scratch[:cnt].copy_(buf, non_blocking=True)
                        dst[lo:lo + cnt].copy_(scratch[:cnt])
                    done[slot] = torch.cuda.Event()
                    done[slot].record(stream)
                k += 1
            out.append(dst)
        if fh.read(1):
            raise ValueError(f"{path}: trailing bytes after data section")
        torch.cuda.current_stream(device).wait_stream(stream)
        stream.synchronize()
    return DeviceBatch(etype, problem, int(n), layout, out[0], out[1])


# ---------------------------------------------------------------------------
# descriptor plumbing
# ---------------------------------------------------------------------------

def _desc_struct(desc: KernelDescriptor, layout: BatchLayout, n: int, base: int, dtype_code: int,
                 geometry: int, coefficients: int, stiffness: int, load: int, error_key: int,
                 out_layout: BatchLayout | None = None, tile: int = 0, ctas_per_sm: int = 0) -> _native.BatchDesc:
    """C descriptor; ``out_layout`` set -> packed output rows in that layout; ``tile`` /
    ``ctas_per_sm``: the tuner's launch knobs (0 = the kernel's own choice)."""
    d = _native.BatchDesc()
    d.element = _native.ELEMENT[desc.element.value]
    d.problem = _native.PROBLEM[desc.problem.value]
    d.variant = _native.VARIANT[desc.variant.value]
    d.geometry_path = _native.GEO_PATH[desc.geometry_path.value]
    d.dtype = dtype_code
    d.layout = _native.LAYOUT[layout.kind.value]
    d.lane_width = layout.lane_width if layout.kind is LayoutKind.LANE_INTERLEAVED else 1
    d.n_elements = n
    d.base_index = base
    d.geometry, d.coefficients = geometry, coefficients
    d.stiffness, d.load, d.error_key = stiffness, load, error_key
    d.tile_elements, d.ctas_per_sm = int(tile), int(ctas_per_sm)
    if out_layout is None:
        d.out_format, d.out_lane_width = _native.OUT_SPLIT, 1
    else:
        d.out_format = _native.OUT_PACKED
        d.out_lane_width = out_layout.lane_width if out_layout.kind is LayoutKind.LANE_INTERLEAVED else 1
    return d


def _traffic(desc: KernelDescriptor, n: int) -> TrafficCounters:
    ns = desc.element.n_shape
    return TrafficCounters(n * desc.element.geometry_size, n * desc.problem.coefficient_size(desc.element),
                           n * ns * ns, n * ns)


def _check_match(desc: KernelDescriptor, batch) -> None:
    etype, problem = coerce_element(batch.element_type), coerce_problem(batch.problem)
    if etype is not desc.element or problem is not desc.problem:
        raise _errors.ShapeMismatch(f"descriptor ({desc.element.value}, {desc.problem.value}) does not match "
                            f"batch ({etype.value}, {problem.value})")


_KIND_TEXT = {
    _native.KIND_DEGENERATE: lambda det, tol: f"|det J| = {abs(det):.3e} <= {tol:.3e}",
    _native.KIND_INVERTED: lambda det, tol: f"det J = {det:.3e} < 0",
}


def _raise_geometry(key, detail) -> None:
    """Raise the reference's exception for an error key, or an (element, point, kind) triple."""
    element, point, kind = _native.decode_error(key) if isinstance(key, int) else key
    if kind == _native.KIND_PIPELINE_TIMEOUT:
        raise NativeLibraryError("integration kernel pipeline timed out (internal error)")
    det, tol = detail(element, point)
    exc = _errors.DegenerateElement if kind == _native.KIND_DEGENERATE else _errors.InvertedElement
    raise exc(_KIND_TEXT[kind](det, tol), element, point)


def _worker_rule_error(desc: KernelDescriptor, geometry_rows, dtype_code: int, n: int, workers: int,
                       base_index: int, stream: int):
    """First error under the reference's ``workers > 1`` rule (``batched.py:569-599``).

    ``geometry_rows``: element-major (n, DS) CUDA tensor.  Each worker range
    [lo, hi) of ``np.linspace(0, n, workers + 1)`` is classified exactly
    (``fek_classify``) with its own block origin (``_run_range`` counts 8192-element
    blocks from ``lo``); the worker error with the smallest element index wins.
    Returns (element, point, kind) or None.
    """
    import torch

    lib = _native.load()
    bounds = np.linspace(0, n, workers + 1).astype(int)
    keys = torch.full((workers,), -1, dtype=torch.int64, device=geometry_rows.device)
    for w, (lo, hi) in enumerate(zip(bounds[:-1], bounds[1:])):
        if hi <= lo:
            continue
        d = _desc_struct(desc, ELEMENT_MAJOR, int(hi - lo), 0, dtype_code, geometry_rows[int(lo)].data_ptr(), 0, 0,
                         0, keys[w].data_ptr())
        _native.check(lib.fek_classify(ctypes.byref(d), stream), "fek_classify")
    found = []
    for w, key in enumerate(keys.tolist()):
        key &= _native.NO_ERROR
        if key != _native.NO_ERROR:
            e, q, k = _native.decode_error(key)
            found.append((int(bounds[w]) + e + base_index, q, k))
    return min(found, key=lambda t: t[0]) if found else None


def _device_error_detail(dd: _native.BatchDesc, local: int, point, stream) -> tuple[float, float]:
    import torch

    out = torch.empty(2, dtype=torch.float64, device="cuda")
    lib = _native.load()
    _native.check(lib.fek_error_detail(ctypes.byref(dd), local, -1 if point is None else point, out.data_ptr(),
                                       stream), "fek_error_detail")
    torch.cuda.current_stream().synchronize()
    det, tol = out.tolist()
    return det, tol


def _packed_views(flat, n: int, ns: int, out_layout: BatchLayout):
    """(stiffness, load) zero-copy views of element-major packed rows, else (None, None)."""
    if out_layout.kind is LayoutKind.LANE_INTERLEAVED and out_layout.lane_width > 1:
        return None, None
    rows = flat.reshape(n, ns * ns + ns)
    A, b = rows[:, : ns * ns], rows[:, ns * ns:]
    if _is_torch(A):
        return A.unflatten(1, (ns, ns)), b
    return A.reshape(n, ns, ns), b


# ---------------------------------------------------------------------------
# device path
# ---------------------------------------------------------------------------

_QUEUES: dict = {}


def _tile_queue(dev, stream: int):
    """Two zeroed int64 words per (device, stream): the kernel's dynamic tile queue.

    Launches on one stream run in order and the last CTA of each launch resets
    the words, so one buffer serves every launch on that stream.
    """
    import torch

    key = (dev.index, stream)
    with _stream_lock:
        q = _QUEUES.get(key)
        if q is None:
            q = _QUEUES[key] = torch.zeros(2, dtype=torch.int64, device=dev)
    return q


def _check_out(out, batch: DeviceBatch, ns: int, packed: bool):
    """Validate caller-supplied outputs before their pointers reach the kernel."""
    import torch

    if packed:
        raise ValueError("out= cannot be combined with packed=True (the packed array is allocated here)")
    if not isinstance(out, (tuple, list)) or len(out) != 2:
        raise TypeError("out must be a pair (stiffness, load) of CUDA tensors")
    n = batch.n_elements
    for name, t, shape in (("stiffness", out[0], (n, ns, ns)), ("load", out[1], (n, ns))):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"out {name} must be a CUDA tensor")
        if t.device != batch.geometry_data.device:
            raise ValueError(f"out {name} is on {t.device}, the batch on {batch.geometry_data.device}")
        if t.dtype != batch.dtype:
            raise TypeError(f"out {name} is {t.dtype}, the batch {batch.dtype}")
        if tuple(t.shape) != shape:
            raise ValueError(f"out {name} must have shape {shape}, got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ValueError(f"out {name} must be contiguous")
        if n and t.data_ptr() % 16:
            raise ValueError(f"out {name} storage must be 16-byte aligned")
    return out[0], out[1]


def _integrate_device(desc: KernelDescriptor, batch: DeviceBatch, out_layout, check: bool, base_index: int,
                      out=None, packed: bool = False, workers: int = 1, tile: int = 0,
                      ctas_per_sm: int = 0) -> BatchResult:
    import torch

    lib = _native.load()
    n, ns = batch.n_elements, desc.element.n_shape
    dev = batch.geometry_data.device
    dtype_code = _native.DTYPE["float64" if batch.dtype == torch.float64 else "float32"]
    olayout = coerce_layout(out_layout)
    flat = None
    if packed:
        if out is not None:
            _check_out(out, batch, ns, packed)
        flat = torch.empty(flat_length(n, ns * ns + ns, olayout), dtype=batch.dtype, device=dev)
        A, b = _packed_views(flat, n, ns, olayout)
        ptr_a, ptr_b = flat.data_ptr(), 0
    else:
        if out is None:
            A = torch.empty((n, ns, ns), dtype=batch.dtype, device=dev)
            b = torch.empty((n, ns), dtype=batch.dtype, device=dev)
        else:
            A, b = _check_out(out, batch, ns, packed)
        ptr_a, ptr_b = A.data_ptr(), b.data_ptr()
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    dd = _desc_struct(desc, batch.layout, n, base_index, dtype_code, batch.geometry_data.data_ptr(),
                      batch.coefficient_data.data_ptr(), ptr_a, ptr_b, err.data_ptr(),
                      out_layout=olayout if packed else None, tile=tile, ctas_per_sm=ctas_per_sm)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        if torch.cuda.is_current_stream_capturing():
            # CUDA-graph capture: a queue of the graph's own (zeroed on every
            # replay by the captured fill), kept alive by the result
            queue = torch.zeros(2, dtype=torch.int64, device=dev)
            if check:
                raise RuntimeError("integrate_batch inside CUDA-graph capture needs check=False "
                                   "(read result.error_word after replay)")
        else:
            queue = _tile_queue(dev, stream)
        dd.scheduler = queue.data_ptr()
        _native.check(lib.fek_integrate(ctypes.byref(dd), stream), "fek_integrate")
        result = BatchResult(desc, n, A, b, _traffic(desc, n), olayout, flat)
        result.error_word = err
        result._queue = queue
        result._launch = (dd, stream, base_index)
        if check:
            key = resolve_error_key(dd, err, stream)
            if key != _native.NO_ERROR:
                detail = lambda e, q: _device_error_detail(dd, e - base_index, q, stream)  # noqa: E731
                if workers > 1:
                    rows = batch if batch.layout.block == 1 else batch.convert(ELEMENT_MAJOR)
                    geo = rows.geometry_data.view(n, desc.element.geometry_size)
                    key = _worker_rule_error(desc, geo, dtype_code, n, workers, base_index, stream)
                _raise_geometry(key, detail)
    return result


def resolve_error_key(dd: _native.BatchDesc, err, stream: int) -> int:
    """The reference's first-error key from a launch's error word (synchronises).

    The kernels decide geometry classes on their own FMA det against 16x the
    tolerance and report ``KIND_NEAR`` for anything closer (never on a valid
    mesh); the exact pass ``fek_classify`` then re-derives the key with the
    reference's rounding (``batched.py:151-177``).
    """
    key = int(err.item()) & _native.NO_ERROR
    if key != _native.NO_ERROR and (key & 127) == _native.KIND_NEAR:
        err.fill_(-1)
        d = _native.BatchDesc.from_buffer_copy(dd)
        d.error_key = err.data_ptr()
        _native.check(_native.load().fek_classify(ctypes.byref(d), stream), "fek_classify")
        key = int(err.item()) & _native.NO_ERROR
    return key


# ---------------------------------------------------------------------------
# host path: chunked H2D -> kernel -> D2H pipeline inside libfek
# ---------------------------------------------------------------------------

_stream_cache: dict[tuple, list] = {}
_stream_lock = threading.Lock()


def _host_streams(device: int):
    """The host pipeline's CUDA streams for this (device, host thread): concurrent integrate_batch
    calls from several threads (the API is re-entrant, batched.py's contract) get their own."""
    import torch

    key = (device, threading.get_ident())
    with _stream_lock:
        if key not in _stream_cache:
            _stream_cache[key] = [torch.cuda.Stream(device=device) for _ in range(HOST_STREAMS)]
        return _stream_cache[key]


def host_chunk_elements(n: int) -> int:
    """Pipeline chunk: ~8+ chunks for big batches (at most 1 Mi elements: C5's 32M-element batches
    ran 379 ms per step at 1 Mi vs 428 ms at 512 Ki on one box, tools/e2e_pageable.py), a
    multiple of 256 elements (every tile size)."""
    chunk = max(16384, min(1 << 20, -(-n // 8)))
    return -(-chunk // 256) * 256


_staging: dict[tuple, np.ndarray] = {}


def _needs_staging(*arrays) -> bool:
    """A large pageable input: DMA from it would serialise in the driver's own bounce buffers."""
    return any(a.nbytes >= hostmem.PIN_THRESHOLD_BYTES and not hostmem.is_pinned(a) for a in arrays)


def _staging_buffer(device: int, nbytes: int) -> np.ndarray:
    """Page-locked staging for fek_integrate_host_staged, kept per (device, host thread) and grown
    on demand."""
    key = (device, threading.get_ident())
    with _stream_lock:
        buf = _staging.get(key)
        if buf is None or buf.nbytes < nbytes:
            buf = _staging[key] = hostmem.empty(-(-nbytes // 8), pin=True)
        return buf


def _copy_threads() -> int:
    """Host copy threads of the staged pipeline: this rank's share of the host cores, at most 8
    (the cache-resident staging ring is copy-engine-bound beyond that: 452 ms per C5 step at 8
    threads, 458 at 12, 464 at 6; tools/e2e_pageable.py)."""
    import os

    per_node = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    return max(1, min(8, (os.cpu_count() or 1) // per_node))


def _aligned_f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ctypes.data % 16:
        b = hostmem.empty(a.shape)
        b[...] = a
        return b
    return a


def _integrate_host(desc: KernelDescriptor, batch, out_layout, base_index: int, packed: bool = False,
                    workers: int = 1, tile: int = 0, ctas_per_sm: int = 0) -> BatchResult:
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device available (there is no CPU fallback)")
    lib = _native.load()
    layout = coerce_layout(batch.layout)
    n, ns = int(batch.n_elements), desc.element.n_shape
    geo = _aligned_f64(batch.geometry_data)
    cof = _aligned_f64(batch.coefficient_data)
    olayout = coerce_layout(out_layout)
    flat = None
    if packed:
        flat = hostmem.empty(flat_length(n, ns * ns + ns, olayout))
        A, b = _packed_views(flat, n, ns, olayout)
        ptr_a, ptr_b = flat.ctypes.data, 0
    else:
        A = hostmem.empty((n, ns, ns))
        b = hostmem.empty((n, ns))
        ptr_a, ptr_b = A.ctypes.data, b.ctypes.data
    dd = _desc_struct(desc, layout, n, base_index, _native.DTYPE["float64"], geo.ctypes.data, cof.ctypes.data,
                      ptr_a, ptr_b, 0, out_layout=olayout if packed else None, tile=tile, ctas_per_sm=ctas_per_sm)
    device = torch.cuda.current_device()
    streams = _host_streams(device)
    chunk = host_chunk_elements(n)
    ws_bytes = lib.fek_host_workspace_bytes(ctypes.byref(dd), len(streams), chunk)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    # the workspace came from torch's current stream; our streams must see it allocated
    cur = torch.cuda.current_stream(device)
    for s in streams:
        s.wait_stream(cur)
    handles = (ctypes.c_void_p * len(streams))(*[s.cuda_stream for s in streams])
    key = ctypes.c_ulonglong(_native.NO_ERROR)
    if _needs_staging(geo, cof):
        # a caller's pageable arrays (e.g. a feklab ElementBatch): staged through page-locked
        # buffers by host copy threads, overlapped with the DMA and the kernels
        st_bytes = lib.fek_host_staging_bytes(ctypes.byref(dd), len(streams), chunk)
        staging = _staging_buffer(device, st_bytes)
        status = lib.fek_integrate_host_staged(ctypes.byref(dd), ws.data_ptr(), ws_bytes, len(streams), handles,
                                               chunk, staging.ctypes.data, st_bytes, _copy_threads(),
                                               ctypes.byref(key))
    else:
        status = lib.fek_integrate_host(ctypes.byref(dd), ws.data_ptr(), ws_bytes, len(streams), handles, chunk,
                                        ctypes.byref(key))
    for s in streams:
        cur.wait_stream(s)
    if status == _native.ERR_GEOMETRY:
        def detail(element, point):
            # upload only the offending element (element-major row) and evaluate it on the GPU
            w = layout.lane_width if layout.kind is LayoutKind.LANE_INTERLEAVED else 1
            dsg = desc.element.geometry_size
            blk, lane = divmod(element - base_index, w)
            row = np.array(geo[blk * w * dsg + lane: blk * w * dsg + lane + dsg * w: w], dtype=np.float64)
            g = torch.from_numpy(row).to(device)
            d1 = _desc_struct(desc, ELEMENT_MAJOR, 1, element, 0, g.data_ptr(), 0, 0, 0, 0)
            return _device_error_detail(d1, 0, point, cur.cuda_stream)

        found = key.value
        if workers > 1:
            rows = unpack_rows(geo, n, desc.element.geometry_size, layout)
            g = torch.from_numpy(np.ascontiguousarray(rows)).to(device)
            found = _worker_rule_error(desc, g, _native.DTYPE["float64"], n, workers, base_index, cur.cuda_stream)
        _raise_geometry(found, detail)
    _native.check(status, "fek_integrate_host")
    return BatchResult(desc, n, A, b, _traffic(desc, n), olayout, flat)


# ---------------------------------------------------------------------------
# public entry point
# ---------------------------------------------------------------------------

def integrate_batch(desc, batch, out_layout: BatchLayout = ELEMENT_MAJOR, workers: int = 1, *,
                    check: bool = True, base_index: int = 0, out=None, packed: bool = False, tile: int = 0,
                    ctas_per_sm: int = 0) -> BatchResult:
    """Integrate every element of ``batch`` with the kernel named by ``desc``.

    Mirrors ``feklab.kernels.integrate_batch`` (``batched.py:536-606``).
    Extra keyword-only knobs: ``check=False`` skips the device->host read of
    the error word for device batches (``result.error_word`` holds it);
    ``base_index`` offsets reported element indices (sharded batches);
    ``out=(A, b)`` supplies preallocated device outputs; ``packed=True`` has
    the kernel write ``flat_output()``'s packed rows in ``out_layout``
    directly (``result.flat``; no repacking pass); ``tile`` (64/128/256, QSS
    natural-path descriptors) and ``ctas_per_sm`` are the tuner's launch knobs
    (0 = the kernel's own choice; results are bitwise independent of both).
    """
    desc = coerce_descriptor(desc)
    _check_match(desc, batch)
    workers = max(1, min(int(workers), int(batch.n_elements)))  # batched.py:569
    if isinstance(batch, DeviceBatch):
        return _integrate_device(desc, batch, out_layout, check, base_index, out, packed, workers, tile, ctas_per_sm)
    if _is_torch(getattr(batch, "geometry_data", None)):
        raise TypeError("batches of torch tensors must be wrapped in DeviceBatch")
    if out is not None:
        raise TypeError("out= is for device batches (host batches return numpy results)")
    return _integrate_host(desc, batch, out_layout, base_index, packed, workers, tile, ctas_per_sm)



def launch_config(desc, layout: BatchLayout, n: int, dtype: str = "float64", tile: int = 0,
                  ctas_per_sm: int = 0) -> dict:
    """Grid/block/smem/tile that ``fek_integrate`` uses for this case (no launch)."""
    desc = coerce_descriptor(desc)
    lib = _native.load()
    dd = _desc_struct(desc, coerce_layout(layout), n, 0, _native.DTYPE[dtype], 0, 0, 0, 0, 0, tile=tile,
                      ctas_per_sm=ctas_per_sm)
    g, bl, sm, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _native.check(lib.fek_launch_config(ctypes.byref(dd), ctypes.byref(g), ctypes.byref(bl), ctypes.byref(sm),
                                        ctypes.byref(t)), "fek_launch_config")
    return {"grid": g.value, "block": bl.value, "smem_bytes": sm.value, "tile_elements": t.value}
