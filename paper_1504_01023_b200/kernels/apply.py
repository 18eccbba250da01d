"""Consumers of the element matrices fused with the integration.

    y, f = apply_batch(desc, device_batch, element_nodes, x)      # y += A x, f += b (assembled)
    row_ptr, col = csr_pattern(element_nodes, n_nodes)            # the global matrix's sparsity
    values, f = assemble_batch(desc, device_batch, element_nodes, row_ptr, col)   # CSR A, f

The paper stops at the element matrices and leaves their use open: assembly, or "without
assembly, in the so called matrix-free approaches", the output possibly kept
"in registers if e.g. assembly operation is designed as extension of procedures performing
numerical integration".  ``fek_apply`` is that extension: the integration
kernel's A_e and b_e stay in registers and are consumed in place,

    y[node(e, r)] += sum_s A_e[r][s] x[node(e, s)],      f[node(e, r)] += b_e[r],

so a Krylov solver's operator application costs one pass over the element inputs (plus the
connectivity and the gathered x) instead of integrate -> store 36 + 6 reals per element ->
read them back.  ``fek_assemble`` is the other consumer the paper names, assembly: the same
registers scattered into a CSR global matrix (``values[csr(i, j)] += A_e[r][s]``).  The sums use atomicAdd, so the order in which element contributions land --
and the last bits of y and f -- vary between runs; A_e and b_e themselves are bitwise the ones
``integrate_batch`` returns.  There is no CPU path.
"""

from __future__ import annotations

import ctypes

from .. import _native
from ..errors import NativeLibraryError
from ..layout import ELEMENT_MAJOR
from ..problems import coerce_descriptor
from .batched import DeviceBatch, _check_match, _desc_struct, _raise_geometry, _device_error_detail, \
    _tile_queue, resolve_error_key


def apply_batch(desc, batch: DeviceBatch, element_nodes, x, y=None, f=None, *, check: bool = True,
                base_index: int = 0):
    """y += sum_e P_e^T A_e P_e x and f += sum_e P_e^T b_e for a device batch; returns (y, f).

    ``element_nodes``: (n, ns) int32 CUDA tensor of global node numbers (``mesh.element_nodes``);
    ``x``: CUDA vector of the batch's dtype indexed by node; ``y`` / ``f``: accumulators (zeros of
    x's shape when None; pass ``f=False`` to skip the load assembly).  The batch must be
    element-major and the descriptor a QSS natural-path one (geo_linear tets, geo_generic prisms).
    Geometry errors raise exactly as ``integrate_batch``'s.
    """
    import torch

    desc = coerce_descriptor(desc)
    _check_match(desc, batch)
    if not isinstance(batch, DeviceBatch):
        raise TypeError("apply_batch takes a DeviceBatch (inputs in HBM)")
    if batch.layout != ELEMENT_MAJOR:
        raise ValueError("apply_batch needs an element-major batch (DeviceBatch.convert(ELEMENT_MAJOR))")
    n, ns = batch.n_elements, desc.element.n_shape
    dev = batch.geometry_data.device
    if not (isinstance(element_nodes, torch.Tensor) and element_nodes.is_cuda and element_nodes.dtype == torch.int32
            and tuple(element_nodes.shape) == (n, ns) and element_nodes.is_contiguous()):
        raise ValueError(f"element_nodes must be a contiguous ({n}, {ns}) int32 CUDA tensor")
    for name, t in (("x", x),) + (() if y is None else (("y", y),)) + (() if f is None or f is False else (("f", f),)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == batch.dtype and t.dim() == 1
                and t.is_contiguous() and t.device == dev):
            raise ValueError(f"{name} must be a contiguous 1-D CUDA tensor of the batch's dtype on {dev}")
    if n:
        lo, hi = torch.aminmax(element_nodes)
        if int(lo) < 0 or int(hi) >= x.numel() or (y is not None and int(hi) >= y.numel()) or \
                (f is not None and f is not False and int(hi) >= f.numel()):
            raise ValueError(f"element_nodes must lie in [0, {x.numel()}) (got [{int(lo)}, {int(hi)}])")
    if y is None:
        y = torch.zeros_like(x)
    if f is None:
        f = torch.zeros_like(x)
    lib = _native.load()
    dtype_code = _native.DTYPE["float64" if batch.dtype == torch.float64 else "float32"]
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    dd = _desc_struct(desc, ELEMENT_MAJOR, n, base_index, dtype_code, batch.geometry_data.data_ptr(),
                      batch.coefficient_data.data_ptr(), 0, 0, err.data_ptr())
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        dd.scheduler = _tile_queue(dev, stream).data_ptr()
        rc = lib.fek_apply(ctypes.byref(dd), element_nodes.data_ptr(), x.data_ptr(), y.data_ptr(),
                           None if f is False else f.data_ptr(), stream)
        if rc == _native.ERR_ARGUMENT:
            raise NativeLibraryError(f"fek_apply: {desc.short_name()} is not a QSS natural-path descriptor "
                                     "or the batch is not element-major")
        _native.check(rc, "fek_apply")
        if check:
            key = resolve_error_key(dd, err, stream)
            if key != _native.NO_ERROR:
                _raise_geometry(key, lambda e, q: _device_error_detail(dd, e - base_index, q, stream))
    return y, (None if f is False else f)


def csr_pattern(element_nodes, n_nodes: int):
    """(row_ptr, col) int32 CUDA tensors: the CSR sparsity of sum_e P_e^T A_e P_e -- every node
    pair that shares an element, columns sorted within each row (built on the device)."""
    import torch

    nodes = element_nodes.long()
    n, ns = nodes.shape
    keys = (nodes[:, :, None] * n_nodes + nodes[:, None, :]).reshape(-1)
    keys = torch.unique(keys)  # sorted
    rows = keys // n_nodes
    col = (keys - rows * n_nodes).to(torch.int32)
    row_ptr = torch.zeros(n_nodes + 1, dtype=torch.int64, device=nodes.device)
    row_ptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n_nodes), 0)
    if int(row_ptr[-1]) >= 2 ** 31:
        raise ValueError("pattern too large for int32 CSR")
    return row_ptr.to(torch.int32), col


def assemble_batch(desc, batch: DeviceBatch, element_nodes, row_ptr, col, values=None, f=None, *,
                   check: bool = True, base_index: int = 0):
    """values += CSR(sum_e P_e^T A_e P_e) and f += sum_e P_e^T b_e for a device batch.

    ``row_ptr`` / ``col``: the CSR pattern (``csr_pattern``); ``values``: its nnz accumulators
    (zeros when None); ``f``: node-indexed load accumulator (zeros of n_nodes when None, False to
    skip).  Same descriptor / batch rules and errors as ``apply_batch``.  Returns (values, f).
    """
    import torch

    desc = coerce_descriptor(desc)
    _check_match(desc, batch)
    if not isinstance(batch, DeviceBatch):
        raise TypeError("assemble_batch takes a DeviceBatch (inputs in HBM)")
    if batch.layout != ELEMENT_MAJOR:
        raise ValueError("assemble_batch needs an element-major batch (DeviceBatch.convert(ELEMENT_MAJOR))")
    n, ns = batch.n_elements, desc.element.n_shape
    dev = batch.geometry_data.device
    for name, t, dt in (("element_nodes", element_nodes, torch.int32), ("row_ptr", row_ptr, torch.int32),
                        ("col", col, torch.int32)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dt and t.is_contiguous() and t.device == dev):
            raise ValueError(f"{name} must be a contiguous int32 CUDA tensor on {dev}")
    if tuple(element_nodes.shape) != (n, ns):
        raise ValueError(f"element_nodes must have shape ({n}, {ns})")
    n_nodes, nnz = row_ptr.numel() - 1, col.numel()
    if n_nodes < 0 or row_ptr.dim() != 1 or col.dim() != 1:
        raise ValueError("row_ptr and col must be 1-D (row_ptr has n_nodes + 1 entries)")
    # a well-formed CSR structure (the kernel searches it; pairs it lacks are reported below)
    if int(row_ptr[0]) != 0 or int(row_ptr[-1]) != nnz or (n_nodes and bool((row_ptr[1:] < row_ptr[:-1]).any())):
        raise ValueError(f"row_ptr must rise from 0 to nnz = {nnz}")
    if nnz:
        clo, chi = torch.aminmax(col)
        if int(clo) < 0 or int(chi) >= n_nodes:
            raise ValueError(f"col must lie in [0, {n_nodes}) (got [{int(clo)}, {int(chi)}])")
    if n:
        lo, hi = torch.aminmax(element_nodes)
        if int(lo) < 0 or int(hi) >= n_nodes:
            raise ValueError(f"element_nodes must lie in [0, {n_nodes}) (got [{int(lo)}, {int(hi)}])")
    if values is None:
        values = torch.zeros(nnz, dtype=batch.dtype, device=dev)
    if f is None:
        f = torch.zeros(n_nodes, dtype=batch.dtype, device=dev)
    for name, t, size in (("values", values, nnz),) + (() if f is False else (("f", f, n_nodes),)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == batch.dtype and t.dim() == 1
                and t.numel() == size and t.is_contiguous() and t.device == dev):
            raise ValueError(f"{name} must be a contiguous 1-D CUDA tensor of {size} {batch.dtype} on {dev}")
    lib = _native.load()
    dtype_code = _native.DTYPE["float64" if batch.dtype == torch.float64 else "float32"]
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    dd = _desc_struct(desc, ELEMENT_MAJOR, n, base_index, dtype_code, batch.geometry_data.data_ptr(),
                      batch.coefficient_data.data_ptr(), 0, 0, err.data_ptr())
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        dd.scheduler = _tile_queue(dev, stream).data_ptr()
        rc = lib.fek_assemble(ctypes.byref(dd), element_nodes.data_ptr(), row_ptr.data_ptr(), col.data_ptr(),
                              values.data_ptr(), None if f is False else f.data_ptr(), stream)
        if rc == _native.ERR_ARGUMENT:
            raise NativeLibraryError(f"fek_assemble: {desc.short_name()} is not a QSS natural-path descriptor "
                                     "or the batch is not element-major")
        _native.check(rc, "fek_assemble")
        if check:
            raw = int(err.item()) & _native.NO_ERROR
            key = resolve_error_key(dd, err, stream)
            if key == _native.NO_ERROR and raw != _native.NO_ERROR:
                # an earlier NEAR key (resolved: no geometry error) may have hidden a pattern miss
                miss = _first_pattern_miss(element_nodes, row_ptr, col)
                key = _native.NO_ERROR if miss is None else (base_index + miss, None, _native.KIND_PATTERN)
            if key != _native.NO_ERROR:
                element, _, kind = _native.decode_error(key) if isinstance(key, int) else key
                if kind == _native.KIND_PATTERN:
                    raise ValueError(f"the CSR pattern has no entry for a node pair of element {element}; "
                                     "values are incomplete")
                _raise_geometry(key, lambda e, q: _device_error_detail(dd, e - base_index, q, stream))
    return values, (None if f is False else f)


def _first_pattern_miss(element_nodes, row_ptr, col):
    """Smallest local element index with a node pair the CSR pattern lacks, or None (torch, on
    the device; only run on the rare path where a NEAR key could have hidden one)."""
    import torch

    n, ns = element_nodes.shape
    if not n:
        return None
    n_nodes = row_ptr.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n_nodes, device=col.device), (row_ptr[1:] - row_ptr[:-1]).long())
    have = rows * n_nodes + col.long()   # sorted when each row's columns are
    have, _ = torch.sort(have)
    nodes = element_nodes.long()
    want = (nodes[:, :, None] * n_nodes + nodes[:, None, :]).reshape(n, -1)
    pos = torch.searchsorted(have, want).clamp_(max=max(have.numel() - 1, 0))
    ok = (have[pos] == want) if have.numel() else torch.zeros_like(want, dtype=torch.bool)
    bad = (~ok).any(dim=1).nonzero()
    return int(bad[0]) if bad.numel() else None
