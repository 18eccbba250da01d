"""CPU baseline: the oracle port of the reference's integrate_batch on all host cores.

TEST / BASELINE INFRASTRUCTURE ONLY (see numpy_oracle.py).  Used by
``bench.py`` for its ``cpu_baseline`` field and for ``--impl reference``.

The reference itself is a numpy program whose ``workers`` threads contend for
the GIL (its own measurements: workers=1 is fastest).  To give
the CPU arm "all the host threads it can use", this runner starts one process
per core, each running the bitwise-faithful numpy restatement
(``numpy_oracle.integrate``) on a contiguous element range -- the reference's
own worker split (``batched.py:573``) -- writing into named shared memory.
``kind`` is therefore "port": the reference's algorithm and numpy arithmetic,
parallelised across processes instead of GIL-bound threads.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time
from multiprocessing import shared_memory

import numpy as np

from . import numpy_oracle as O

_STATE = {}


class _Shared:
    """A named shared-memory float64 array (the workers attach by name)."""

    def __init__(self, shape, fill=None):
        self.shape = tuple(int(x) for x in shape)
        size = max(int(np.prod(self.shape)) * 8, 8)
        self.shm = shared_memory.SharedMemory(create=True, size=size)
        self.array = np.ndarray(self.shape, dtype=np.float64, buffer=self.shm.buf)
        if fill is None:
            self.array.fill(0.0)  # fault the pages in before timing
        else:
            self.array[...] = fill

    def spec(self):
        return self.shm.name, self.shape

    def close(self):
        self.array = None
        try:
            self.shm.close()
        except BufferError:  # a caller still holds a view; the mapping goes with it
            pass
        self.shm.unlink()


def _attach(name, shape):
    # (forkserver workers share the parent's resource tracker, which the
    # parent's unlink() settles; attaching re-registers the same name)
    shm = shared_memory.SharedMemory(name=name)
    return shm, np.ndarray(shape, dtype=np.float64, buffer=shm.buf)


def _init_worker(config, specs):
    _STATE.clear()
    _STATE.update(config)
    _STATE["_shm"] = []
    for key, (name, shape) in specs.items():
        shm, arr = _attach(name, shape)
        _STATE["_shm"].append(shm)
        _STATE[key] = arr


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
    """Process pool holding one workload; ``run(lo, hi)`` integrates a range in parallel.

    Workers come from a ``forkserver`` (a clean single-threaded parent), not
    a fork of this process -- which may hold CUDA and torch threads -- and
    see the inputs and outputs through named shared memory.
    """

    def __init__(self, variant, path, problem, etype, geo_rows, coef_rows, processes: int | None = None):
        self.processes = processes or os.cpu_count() or 1
        ns = 4 if etype == O.TET else 6
        n = geo_rows.shape[0]
        config = dict(variant=variant, path=path, problem=problem, etype=etype)
        self._arrays = {"geo": _Shared(geo_rows.shape, geo_rows), "coef": _Shared(coef_rows.shape, coef_rows),
                        "A": _Shared((n, ns, ns)), "b": _Shared((n, ns))}
        self.A, self.b = self._arrays["A"].array, self._arrays["b"].array
        specs = {k: v.spec() for k, v in self._arrays.items()}
        if self.processes > 1:
            self._pool = mp.get_context("forkserver").Pool(self.processes, initializer=_init_worker,
                                                           initargs=(config, specs))
        else:
            self._pool = None
            _init_worker(config, specs)

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
        for shm in _STATE.pop("_shm", []):
            shm.close()
        _STATE.clear()
        self.A = self.b = None
        for arr in self._arrays.values():
            arr.close()
        self._arrays = {}

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
