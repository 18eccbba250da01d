"""Timing harness, layout tuner and run reporting on the GPU.

Mirror of ``pkg/src/feklab/bench.py``: the same ``RunRecord``, CSV columns
(``bench.py:36-52``, so the reference's ``report/`` charts read the output
unchanged), ``run_benchmark`` / ``tune`` signatures and enumeration order,
and the counter check before timing (``bench.py:116-124``).

What changes is where the time goes.  By default (``inputs="device"``) a
host batch is uploaded to HBM once before timing, as the paper times its
kernels (``PAPER.md:889-895``), and each repeat is one stream-ordered
``integrate_batch`` call on the resident ``DeviceBatch`` timed with CUDA
events into preallocated outputs; the per-element time is the kernel's.
``inputs="host"`` times the whole public call on host arrays (H2D + kernel +
D2H) with the wall clock instead.  An injected ``clock`` (the reference's
deterministic-test hook) always selects wall-clock timing, with a device
synchronize before each reading.

``workers`` keeps its column and is passed through to ``integrate_batch``,
which runs every batch on the current GPU.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass
from statistics import median

from .errors import CounterMismatch
from .kernels import DeviceBatch, global_accesses, integrate_batch
from .layout import LANE_WIDTHS, BatchLayout, ElementBatch, LayoutKind, convert
from .perfmodel import ProcessorProfile, efficiency, kernel_cost, time_bound
from .problems import KernelDescriptor


def default_worker_counts() -> tuple[int, ...]:
    """{1, physical cores, 2 x cores} (``bench.py:23-33``); kept for the CLI's ``tune`` default."""
    try:
        import psutil

        cores = psutil.cpu_count(logical=False) or 1
    except ImportError:  # pragma: no cover
        import os

        cores = os.cpu_count() or 1
    return tuple(sorted({1, cores, 2 * cores}))


CSV_COLUMNS = ("variant", "geo", "element", "problem", "layout", "lane_width", "workers", "n_elements",
               "ns_per_element", "ns_mad", "accesses_per_element", "ops_model", "intensity", "bound_ns",
               "efficiency_pct")

TUNE_TIME_FLOOR_MS = 10.0


def fixed(x: float, digits: int, like: float | None = None) -> str:
    """The reference's fixed-point format (``bench.py:80-90``), with two more digits below 1 ns.

    B200 times and bounds are fractions of a nanosecond per element, where
    ``.2f`` / ``.3f`` would keep only one or two significant digits.  ``like``
    picks the digit count from another value (the MAD follows its median).
    """
    ref = x if like is None else like
    return f"{x:.{digits if abs(ref) >= 1.0 else digits + 2}f}"


@dataclass(frozen=True)
class RunRecord:
    """One timed configuration with its cost-model context (``bench.py:58-92``)."""

    descriptor: KernelDescriptor
    layout: BatchLayout
    n_elements: int
    ns_per_element: float
    ns_mad: float
    measured_accesses: float
    model_bound_ns: float
    efficiency_pct: int
    worker_count: int
    verified: bool = True

    def csv_row(self) -> list[str]:
        cost = kernel_cost(self.descriptor)
        d = self.descriptor
        return [d.variant.value, d.geometry_path.value, d.element.value, d.problem.value,
                self.layout.kind.value, str(self.layout.lane_width), str(self.worker_count), str(self.n_elements),
                fixed(self.ns_per_element, 3), fixed(self.ns_mad, 3, like=self.ns_per_element), f"{self.measured_accesses:.0f}",
                str(cost.op_count), str(cost.arithmetic_intensity), fixed(self.model_bound_ns, 2),
                str(self.efficiency_pct)]


def _sync():
    import torch

    if torch.cuda.is_available():
        torch.cuda.synchronize()


def _device_times(desc, batch: DeviceBatch, workers: int, repeats: int) -> list[float]:
    """Per-repeat kernel time in ns/element: CUDA events on the launching stream, resident outputs."""
    import torch

    n, ns = batch.n_elements, batch.element_type.n_shape
    dev = batch.geometry_data.device
    A = torch.empty((n, ns, ns), dtype=batch.dtype, device=dev)
    b = torch.empty((n, ns), dtype=batch.dtype, device=dev)
    out = []
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream()
        for _ in range(repeats):
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # an untimed call first keeps the stream busy while the timed call is prepared on
            # the host, so the events bracket the launch itself (not the Python call overhead)
            integrate_batch(desc, batch, workers=workers, check=False, out=(A, b))
            start.record(stream)
            integrate_batch(desc, batch, workers=workers, check=False, out=(A, b))
            stop.record(stream)
            stop.synchronize()
            out.append(start.elapsed_time(stop) * 1e6 / n)
        # surface a geometry error of the timed launches (the warm-up already checked the same input)
        integrate_batch(desc, batch, workers=workers, out=(A, b))
    return out


def run_benchmark(batch, desc: KernelDescriptor, profile: ProcessorProfile, layout: BatchLayout | None = None,
                  workers: int = 1, repeats: int = 5, clock=None, verified: bool = True,
                  inputs: str = "device") -> RunRecord:
    """Median-of-repeats timing of one configuration (``bench.py:95-147``).

    The batch is converted to ``layout`` first when given.  ``batch`` may be a
    host ``ElementBatch`` or a ``DeviceBatch``; ``inputs`` selects whether a
    host batch is made resident first ("device") or timed through the host
    call ("host").
    """
    if repeats < 3:
        raise ValueError("need at least 3 repeats for a meaningful median")
    if inputs not in ("device", "host"):
        raise ValueError(f"inputs must be 'device' or 'host', got {inputs!r}")
    if layout is not None and layout != batch.layout:
        batch = convert(batch, layout)
    layout = batch.layout
    n = batch.n_elements
    if inputs == "device" and isinstance(batch, ElementBatch):
        batch = DeviceBatch.from_host(batch)

    # warm-up doubles as the counter check (and raises geometry errors)
    result = integrate_batch(desc, batch, workers=workers)
    measured = result.traffic.per_element(n)
    model = global_accesses(desc.element, desc.problem)
    if measured != model:
        raise CounterMismatch(f"{desc.short_name()}: measured {measured} global accesses per element, "
                              f"cost model says {model}")
    del result

    if clock is None and isinstance(batch, DeviceBatch):
        times = _device_times(desc, batch, workers, repeats)
    else:
        clock = clock or time.perf_counter
        times = []
        for _ in range(repeats):
            _sync()
            t0 = clock()
            integrate_batch(desc, batch, workers=workers)
            _sync()
            times.append((clock() - t0) * 1e9 / n)
    med = median(times)
    mad = median(abs(t - med) for t in times)
    if med <= 0:
        raise RuntimeError("non-positive median time; clock is broken")
    bound = time_bound(desc, profile)
    return RunRecord(desc, layout, n, med, mad, measured, bound, efficiency(med, bound), workers, verified)


def tune(batch, desc: KernelDescriptor, profile: ProcessorProfile, lane_widths: tuple[int, ...] = LANE_WIDTHS[1:],
         worker_counts: tuple[int, ...] = (1,), repeats: int = 5, clock=None, run_fn=run_benchmark,
         verified: bool = True) -> tuple[RunRecord, list[RunRecord]]:
    """Exhaustive layout x lane width x worker sweep (``bench.py:150-196``).

    Element-major first, then lane-interleaved by ascending width; ascending
    worker count within a layout.  Best = smallest ns/element, first tie kept.
    A ``DeviceBatch`` is re-laid-out in HBM (``fek_convert_layout``); a host
    batch on the host, then uploaded by ``run_benchmark``.
    """
    layouts = [BatchLayout(LayoutKind.ELEMENT_MAJOR)]
    layouts += [BatchLayout(LayoutKind.LANE_INTERLEAVED, w) for w in sorted(lane_widths)]
    records = []
    for lay in layouts:
        converted = convert(batch, lay)
        for workers in worker_counts:
            records.append(run_fn(converted, desc, profile, layout=None, workers=workers, repeats=repeats,
                                  clock=clock, verified=verified))
        del converted
    best = min(records, key=lambda r: r.ns_per_element)
    if best.ns_per_element * batch.n_elements < TUNE_TIME_FLOOR_MS * 1e6:
        warnings.warn(f"per-run time below the {TUNE_TIME_FLOOR_MS:.0f} ms timing floor; "
                      "increase the batch size for trustworthy tuning", stacklevel=2)
    return best, records


def format_records(records, fmt: str = "table", unverified: bool = False) -> str:
    """CSV or right-aligned table, input order kept (``bench.py:199-223``)."""
    if not records:
        raise ValueError("no records to report")
    rows = [r.csv_row() for r in records]
    head = "# UNVERIFIED: correctness gate was skipped\n" if unverified else ""
    if fmt == "csv":
        return head + "\n".join([",".join(CSV_COLUMNS)] + [",".join(r) for r in rows]) + "\n"
    if fmt != "table":
        raise ValueError(f"unknown format {fmt!r}")
    shown = [r[:-1] + [r[-1] + "%"] for r in rows]
    widths = [max(len(h), *(len(r[i]) for r in shown)) for i, h in enumerate(CSV_COLUMNS)]
    lines = ["  ".join(cell.rjust(w) for cell, w in zip(r, widths)) for r in [list(CSV_COLUMNS)] + shown]
    return head + "\n".join(lines) + "\n"
