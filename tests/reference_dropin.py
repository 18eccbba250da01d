"""pytest plugin: run the REFERENCE's own test suite with the B200 drop-in behind feklab's API.

    python -m pytest baseline/_ref/tests -p reference_dropin      (PYTHONPATH = baseline/_ref:tests:<repo>)

SURVEY.md section 8(c) "Harness": the reference's tests (``pkg/tests/test_kernels.py``,
``test_acceptance.py``, ...) import ``integrate_batch`` / ``integrate_element`` from
``feklab`` / ``feklab.kernels``.  Before any test module is collected, every binding of those
two names in the imported ``feklab`` modules (the package, ``feklab.kernels``,
``feklab.kernels.batched`` / ``scalar``, and the reference's own callers ``feklab.verify``,
``feklab.bench``, ``feklab.cli``) is replaced by ``paper_1504_01023_b200``'s -- so the stock
tests, and the reference's CLI/verify/bench paths they drive, integrate on the GPU through the
C-ABI.  Reference objects (descriptors, ``ElementBatch``, ``ElementGeometry``,
``CoefficientSet``) cross the boundary duck-typed; everything else in feklab (mesh, layout,
oracle, perfmodel) stays the reference's.
"""

from __future__ import annotations

import importlib
import pkgutil
import sys

REPLACED: dict[str, list[str]] = {}
CALLS: dict[str, int] = {}


def _install() -> None:
    import feklab

    import paper_1504_01023_b200 as fek
    from paper_1504_01023_b200 import _native

    _native.load()  # fails loudly without libfek.so: no CPU fallback

    originals = {}
    for info in pkgutil.walk_packages(feklab.__path__, "feklab."):
        if info.name.startswith("feklab.report"):
            continue
        importlib.import_module(info.name)
    from feklab.kernels import batched, scalar

    import feklab.errors

    fek.errors.bind_exception_types(feklab.errors)  # raise feklab's own exception classes
    originals["integrate_batch"] = batched.integrate_batch
    originals["integrate_element"] = scalar.integrate_element
    def counted(fn, name):
        def call(*a, **k):
            CALLS[name] = CALLS.get(name, 0) + 1
            return fn(*a, **k)
        call.__wrapped__ = fn
        call.__name__ = call.__qualname__ = fn.__name__
        call.__doc__ = fn.__doc__
        return call

    ours = {n: counted(getattr(fek, n), n) for n in ("integrate_batch", "integrate_element")}
    for name, mod in list(sys.modules.items()):
        if not (name == "feklab" or name.startswith("feklab.")) or mod is None:
            continue
        for attr, orig in originals.items():
            if getattr(mod, attr, None) is orig:
                setattr(mod, attr, ours[attr])
                REPLACED.setdefault(attr, []).append(name)


def pytest_configure(config):
    _install()


def pytest_report_header(config):
    import paper_1504_01023_b200._native as nat

    return [f"reference_dropin: feklab integrate_batch/integrate_element -> paper_1504_01023_b200 "
            f"({nat.LIB_PATH}); rebound in {sorted(set(m for v in REPLACED.values() for m in v))}"]


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"reference_dropin: GPU drop-in calls {dict(sorted(CALLS.items()))}")
