"""The CPU oracle is pinned to the reference before it is trusted.

Every golden array was produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce the reference's
batched kernels BIT FOR BIT on all 18 descriptors, its first-error rule, and
agree with the reference's Algorithm-1 / refined-rule oracles.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import numpy_oracle as O

CASES = [("tet", "poisson"), ("prism", "poisson"), ("tet", "convdiff"), ("prism", "convdiff")]


def _descriptors(et):
    paths = ("linear", "generic") if et == "tet" else ("generic",)
    return [(v, p) for v in ("qss", "sqs", "ssq") for p in paths]


@pytest.mark.parametrize("et,pb", CASES)
def test_oracle_bitwise_equals_reference_batched(et, pb):
    z = golden(f"corpus_{et}_{pb}.npz")
    for v, p in _descriptors(et):
        A, b = O.integrate(v, p, pb, et, z["geometry_rows"], z["coefficient_rows"])
        name = f"{v}_{p}_{et}_{pb}"
        assert np.array_equal(A, z[f"A_{name}"]), name
        assert np.array_equal(b, z[f"b_{name}"]), name


@pytest.mark.parametrize("et,pb", CASES)
def test_oracle_matches_algorithm1(et, pb):
    z = golden(f"corpus_{et}_{pb}.npz")
    A, b = O.integrate("qss", O.natural_path(et), pb, et, z["geometry_rows"], z["coefficient_rows"])
    assert O.rel_frobenius(A, z["A_algorithm1"]).max() < 1e-12
    assert O.rel_frobenius(b, z["b_algorithm1"]).max() < 1e-12


def test_oracle_tables_bitwise():
    r = golden("refelem.npz")
    for et in ("tet", "prism"):
        w, vals, ld = O.tables(et)
        assert np.array_equal(w, r[f"{et}_weights"])
        assert np.array_equal(vals, r[f"{et}_values"])
        assert np.array_equal(ld, r[f"{et}_local_derivatives"])


def test_oracle_twisted_prisms_vs_refined_rule():
    z = golden("twisted_prisms.npz")
    for pb, rows in (("convdiff", z["convdiff_rows"]), ("poisson", z["poisson_rows"])):
        for v in ("qss", "sqs", "ssq"):
            A, b = O.integrate(v, "generic", pb, "prism", z["geometry_rows"], rows)
            assert O.rel_frobenius(A, z[f"A_{pb}"]).max() < 1e-10
            assert O.rel_frobenius(b, z[f"b_{pb}"]).max() < 1e-10


def _error_cases():
    z = golden("errors.npz")
    names = sorted({k.split("__")[0] for k in z.files if "__" in k})
    return z, names


def block_rule_rows():
    """Same formula as tests/golden/make_golden.py:block_rule_rows."""
    z = golden("errors.npz")
    good = np.array([(0, 0, -1), (1, 0, -1), (0, 1, -1), (0, 0, 1), (1, 0, 1), (0, 1, 1)], dtype=float)
    n = 8300
    rows = np.tile(good.reshape(-1), (n, 1))
    rows[:, 0::3] += 1e-3 * np.arange(n)[:, None]
    rows[100] = z["prism_partly_inverted"].reshape(-1)
    rows[8200] = -good.reshape(-1)
    return rows, np.zeros((n, 20))


def error_case_inputs(z, name):
    if name == "prism_block_rule":
        return block_rule_rows()
    return z[f"{name}__geometry_rows"], z[f"{name}__coefficient_rows"]


def test_oracle_first_error_rule():
    z, names = _error_cases()
    checked = 0
    for name in names:
        if name == "prism_partly_inverted":
            continue
        geo, cof = error_case_inputs(z, name)
        et = "tet" if name.startswith("tet") else "prism"
        pb = "poisson" if cof.shape[1] in (4, 6) else "convdiff"
        for v, p in _descriptors(et):
            want = z[f"{name}__{v}_{p}_{et}_{pb}"]
            with pytest.raises(O.OracleGeometryError) as err:
                O.integrate(v, p, pb, et, geo, cof)
            kind = 1 if err.value.kind == "degenerate" else 2
            point = -1 if err.value.point_index is None else err.value.point_index
            assert (kind, err.value.element_index, point) == tuple(want), (name, v, p)
            checked += 1
    assert checked >= 20


def boundary_fixtures():
    """(et, j, geometry rows, {descriptor short name: (kind, element, point)}) of boundary.npz."""
    z = golden("boundary.npz")
    for et in ("tet", "prism"):
        geo = z[f"{et}_geometry"]
        for j in range(geo.shape[0]):
            want = {k.split("__")[1]: tuple(int(x) for x in z[k]) for k in z.files if k.startswith(f"{et}_{j}__")}
            yield et, j, geo[j], want


def test_oracle_classification_at_the_tolerance_boundary():
    """|det J| within ~1e-3 (and within ulps) of 1e-14 diag^3: bitwise the reference's verdicts.

    The fixtures hold elements whose bounding-box cube is host-independent (make_golden.py
    boundary_cases), so the oracle's own numpy `scale**3` reproduces the reference's here too.
    """
    checked = errors = 0
    for et, j, geo, want in boundary_fixtures():
        for name, code in want.items():
            v, p = name.split("_")[:2]
            pb = name.split("_")[-1]
            cof = np.ones((3, (4 if et == "tet" else 6) if pb == "poisson" else 20))
            try:
                O.integrate(v, p, pb, et, geo, cof)
                got = (0, -1, -1)
            except O.OracleGeometryError as err:
                got = (1 if err.kind == "degenerate" else 2, err.element_index,
                       -1 if err.point_index is None else err.point_index)
                errors += 1
            assert got == code, (et, j, name)
            checked += 1
    assert checked >= 800 and errors >= 400
