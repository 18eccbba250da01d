"""CPU baseline: the oracle port of the reference's integrate_batch on all host cores.

TEST / BASELINE INFRASTRUCTURE ONLY (see numpy_oracle.py).  Used by
``bench.py`` for its ``cpu_baseline`` field and for ``--impl reference``.

The reference itself is a numpy program whose ``workers`` threads contend for
the GIL (its own measurements: workers=1 is fastest).  To give
the CPU arm "all the host threads it can use", this runner forks one process
per core, each running the bitwise-faithful numpy restatement
(``numpy_oracle.integrate``) on a contiguous element range -- the reference's
own worker split (``batched.py:573``) -- writing into shared anonymous
memory.  ``kind`` is therefore "port": the reference's algorithm and numpy
arithmetic, parallelised across processes instead of GIL-bound threads.
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os
import time

import numpy as np

from . import numpy_oracle as O

_STATE = {}


def _shared(shape) -> np.ndarray:
    size = int(np.prod(shape)) * 8
    buf = mmap.mmap(-1, max(size, 8))
    arr = np.frombuffer(buf, dtype=np.float64, count=int(np.prod(shape))).reshape(shape)
    arr.fill(0.0)  # fault the pages in before forking, so timed runs measure compute only
    return arr


def _work(args):
    lo, hi = args
    s = _STATE
    if hi <= lo:
        return 0
    A, b = O.integrate(s["variant"], s["path"], s["problem"], s["etype"], s["geo"][lo:hi], s["coef"][lo:hi])
    s["A"][lo:hi] = A
    s["b"][lo:hi] = b
    return hi - lo


class PortPool:
    """Fork pool holding one workload; ``run(lo, hi)`` integrates a range in parallel."""

    def __init__(self, variant, path, problem, etype, geo_rows, coef_rows, processes: int | None = None):
        self.processes = processes or os.cpu_count() or 1
        ns = 4 if etype == O.TET else 6
        n = geo_rows.shape[0]
        _STATE.clear()
        _STATE.update(variant=variant, path=path, problem=problem, etype=etype,
                      geo=np.ascontiguousarray(geo_rows), coef=np.ascontiguousarray(coef_rows),
                      A=_shared((n, ns, ns)), b=_shared((n, ns)))
        self.A, self.b = _STATE["A"], _STATE["b"]
        self._pool = mp.get_context("fork").Pool(self.processes) if self.processes > 1 else None

    def run(self, lo: int, hi: int) -> float:
        """Integrate elements [lo, hi); returns wall seconds."""
        p = self.processes
        bounds = np.linspace(lo, hi, p + 1).astype(int)
        ranges = list(zip(bounds[:-1], bounds[1:]))
        t0 = time.perf_counter()
        if self._pool is None:
            for r in ranges:
                _work(r)
        else:
            self._pool.map(_work, ranges, chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        if self._pool is not None:
            self._pool.close()
            self._pool.join()
            self._pool = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def cpu_cores() -> dict:
    try:
        import psutil

        return {"logical": psutil.cpu_count(logical=True), "physical": psutil.cpu_count(logical=False)}
    except Exception:
        return {"logical": os.cpu_count(), "physical": None}
