"""The REFERENCE's own test suite, run against the B200 drop-in (SURVEY.md section 8(c) "Harness").

``baseline/_ref`` holds the stock reference (``pip install --target baseline/_ref`` of
``/root/reference/pkg``, plus its ``tests/`` directory; ``__graft_entry__.build()`` creates it
when ``/root/reference`` is present -- it is git-ignored and travels to the GPU box with the
snapshot).  The ``reference_dropin`` plugin rebinds feklab's ``integrate_batch`` /
``integrate_element`` to ``paper_1504_01023_b200``'s before collection, so every test that
integrates -- ``test_kernels.py:56-341``, ``test_acceptance.py:96-305`` and the CLI / verify /
bench paths they drive -- runs on the GPU through the C-ABI.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
MODULES = ["test_kernels.py", "test_acceptance.py", "test_geometry.py", "test_layout.py", "test_mesh.py",
           "test_oracle.py", "test_perfmodel.py", "test_refelem.py", "test_bench_cli.py"]


def _run(modules, extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests"), ROOT])
    cmd = [sys.executable, "-m", "pytest", "-p", "reference_dropin", "-p", "no:cacheprovider",
           "--rootdir", os.path.join(REF, "tests"), *extra, *[os.path.join(REF, "tests", m) for m in modules]]
    return subprocess.run(cmd, cwd=os.path.join(REF, "tests"), env=env, capture_output=True, text=True,
                          timeout=1800)


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                    reason="baseline/_ref (stock reference + its tests) not installed in this snapshot")
def test_reference_suite_passes_on_the_gpu_dropin():
    res = _run(MODULES)
    tail = (res.stdout + res.stderr)[-6000:]
    assert res.returncode == 0, tail
    m = re.search(r"(\d+) passed", res.stdout)
    assert m and int(m.group(1)) >= 190, tail
    assert "reference_dropin: feklab integrate_batch/integrate_element -> paper_1504_01023_b200" in res.stdout
    assert "libfek.so" in res.stdout
    calls = re.search(r"GPU drop-in calls \{'integrate_batch': (\d+), 'integrate_element': (\d+)\}", res.stdout)
    assert calls and int(calls.group(1)) > 300 and int(calls.group(2)) > 1000, tail
