"""GPU classification at the degeneracy bound, against the reference's own verdicts.

`tests/golden/boundary.npz` holds 48 tets and 48 prisms whose |det J| lies within ~1e-3 of
the tolerance 1e-14 diag^3 (half of the tets within a few ulps of it), each the middle
element of a 3-element batch, with the reference's `integrate_batch` verdict for every
descriptor (make_golden.py boundary_cases).  About half of them were classified differently
by the round-1 kernels (FMA det, twice-rounded tol).  The kernels now flag every point within
16 tol as NEAR and `fek_classify` re-derives the key with the reference's rounding
(batched.py:136-177); outputs of such ill-conditioned elements are not compared, only the
error semantics (kind, element, point, message) -- bit-exact index work.
"""

import numpy as np
import pytest

import paper_1504_01023_b200 as fek
from conftest import GOLDEN, golden
from paper_1504_01023_b200 import (DeviceBatch, ElementBatch, ElementType, GeometryPath, KernelDescriptor,
                                   ProblemClass, Variant, integrate_batch)
from test_oracle import boundary_fixtures

pytestmark = pytest.mark.gpu

ET = {"tet": ElementType.TETRAHEDRON, "prism": ElementType.PRISM}
PB = {"poisson": ProblemClass.POISSON, "convdiff": ProblemClass.CONV_DIFF}


def _desc(short_name):
    v, p, et, pb = short_name.split("_")
    return KernelDescriptor(Variant(v), GeometryPath(p), ProblemClass(pb), ElementType(et))


def _verdict(desc, batch):
    desc = _desc(desc) if isinstance(desc, str) else desc
    try:
        integrate_batch(desc, batch)
        return (0, -1, -1), ""
    except fek.GeometryError as err:
        kind = 1 if isinstance(err, fek.DegenerateElement) else 2
        return (kind, err.element_index, -1 if err.point_index is None else err.point_index), str(err)


def _messages():
    lines = open(GOLDEN + "/boundary_messages.tsv").read().strip("\n").split("\n")
    return dict((line.split("\t", 1) + [""])[:2] for line in lines)


def test_boundary_classification_matches_reference_bitwise():
    msgs = _messages()
    checked = 0
    for et, j, geo, want in boundary_fixtures():
        for name, code in want.items():
            pb = name.split("_")[-1]
            cof = np.ones((3, (4 if et == "tet" else 6) if pb == "poisson" else 20))
            host = ElementBatch.from_arrays(ET[et], PB[pb], geo, cof)
            for batch in (host, DeviceBatch.from_host(host)):
                got, msg = _verdict(name, batch)
                assert got == code, (et, j, name, type(batch).__name__)
                assert msg == msgs[f"{et}_{j}__{name}"], (et, j, name)
                checked += 1
    assert checked >= 1700


def test_round1_kernels_would_have_misclassified_some_fixtures():
    z = golden("boundary.npz")
    assert int(z["tet_round1_misclassified"][0]) >= 20 and int(z["prism_round1_misclassified"][0]) >= 20


def _big_batch(et, n, plant):
    """n valid elements (shifted copies of the reference element) with rows planted at given indices."""
    ref = ET[et].reference_vertices.reshape(-1).astype(float)
    rows = np.tile(ref, (n, 1))
    rows[:, 0::3] += 1e-3 * (np.arange(n) % 1000)[:, None]
    for e, row in plant.items():
        rows[e] = row
    return rows


@pytest.mark.parametrize("et", ["tet", "prism"])
def test_near_but_valid_element_does_not_hide_a_later_error(et):
    """The kernel's NEAR key (smaller) must not mask a real error further on; and a batch whose
    only flagged element is valid by the reference's rounding integrates without error."""
    fixtures = list(boundary_fixtures())
    desc = _desc(f"qss_generic_{et}_convdiff")
    valid = next(g[1] for e, j, g, w in fixtures if e == et and w[desc.short_name()] == (0, -1, -1))
    bad = next(g[1] for e, j, g, w in fixtures if e == et and w[desc.short_name()][0] == 2)
    n = 300_000  # several host-pipeline chunks
    cof = np.ones((n, 20))
    rows = _big_batch(et, n, {1000: valid})
    for batch in (ElementBatch.from_arrays(ET[et], PB["convdiff"], rows, cof),):
        for b in (batch, DeviceBatch.from_host(batch)):
            res = integrate_batch(desc, b)
            assert res.n_elements == n
    rows = _big_batch(et, n, {1000: valid, 250_123: bad})
    batch = ElementBatch.from_arrays(ET[et], PB["convdiff"], rows, cof)
    for b in (batch, DeviceBatch.from_host(batch)):
        got, _ = _verdict(desc, b)
        assert got[0] == 2 and got[1] == 250_123, got


def test_device_tolerance_is_the_correctly_rounded_cube():
    """tol = 1e-14 * scale**3 with the cube rounded once (batched.py:167); (s*s)*s differs on ~26%."""
    from fractions import Fraction

    from paper_1504_01023_b200.geometry import ElementGeometry, _device_jacobian

    rng = np.random.default_rng(7)
    naive_differs = 0
    for _ in range(400):
        coords = rng.uniform(-1, 1, (4, 3)) * 10.0 ** rng.uniform(-3, 3)
        span = coords.max(0) - coords.min(0)
        s = float(np.sqrt(((span[0] * span[0]) + span[1] * span[1]) + span[2] * span[2]))
        want = 1e-14 * float(Fraction(s) ** 3)
        _, _, _, tol = _device_jacobian(ElementGeometry(ElementType.TETRAHEDRON, coords), -1)
        assert tol == want
        naive_differs += (1e-14 * ((s * s) * s)) != want
    assert naive_differs > 40


def _workers_rows():
    z = golden("workers.npz")
    good = ElementType.PRISM.reference_vertices.astype(float)
    rows = np.tile(good.reshape(-1), (20000, 1))
    rows[:, 0::3] += 1e-3 * (np.arange(20000) % 1000)[:, None]
    rows[16000] = z["prism_partly_inverted"].reshape(-1)
    rows[16500] = -good.reshape(-1)
    return z, rows


@pytest.mark.parametrize("workers", [1, 2, 3, 7])
def test_workers_first_error_rule_matches_reference(workers):
    """workers > 1: per-range 8192-blocks, then the smallest element over ranges (batched.py:569-599)."""
    from paper_1504_01023_b200.layout import BatchLayout, LayoutKind, convert

    z, rows = _workers_rows()
    for pb in ("poisson", "convdiff"):
        problem = PB[pb]
        cof = np.zeros((rows.shape[0], problem.coefficient_size(ElementType.PRISM)))
        host = ElementBatch.from_arrays(ElementType.PRISM, problem, rows, cof)
        inter = convert(host, BatchLayout(LayoutKind.LANE_INTERLEAVED, 16))
        for name in (f"{v}_generic_prism_{pb}" for v in ("qss", "sqs", "ssq")):
            want = tuple(int(x) for x in z[f"w{workers}__{name}"])
            for batch in (host, DeviceBatch.from_host(host), DeviceBatch.from_host(inter)):
                desc = _desc(name)
                with pytest.raises(fek.InvertedElement) as err:
                    integrate_batch(desc, batch, workers=workers)
                got = (2, err.value.element_index, err.value.point_index)
                assert got == want, (workers, name, type(batch).__name__)
