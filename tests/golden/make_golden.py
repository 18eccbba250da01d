"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The GPU box never runs this (``/root/reference`` does not exist there); the
committed ``.npz`` files travel instead.  Every array below is an output of
the reference's own public functions (``feklab.integrate_batch``,
``feklab.oracle.integrate_reference`` / ``integrate_high_order``,
``feklab.mesh.generate_mesh``, ``feklab.refelem.reference_element``) on
seeded inputs drawn with the reference's own corpus generators
(``feklab.verify.random_geometry`` / ``random_coefficients``).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import feklab  # noqa: E402
from feklab.errors import GeometryError  # noqa: E402
from feklab.geometry import ElementGeometry  # noqa: E402
from feklab.kernels import integrate_batch  # noqa: E402
from feklab.layout import ElementBatch, build_batch  # noqa: E402
from feklab.mesh import MeshSpec, generate_mesh  # noqa: E402
from feklab.oracle import integrate_high_order, integrate_reference  # noqa: E402
from feklab.problems import CoefficientSet, ProblemClass, case_descriptors  # noqa: E402
from feklab.refelem import ElementType, reference_element  # noqa: E402
from feklab.verify import random_coefficients, random_geometry  # noqa: E402

TET, PRISM = ElementType.TETRAHEDRON, ElementType.PRISM
POISSON, CONVDIFF = ProblemClass.POISSON, ProblemClass.CONV_DIFF
CASES = ((TET, POISSON), (PRISM, POISSON), (TET, CONVDIFF), (PRISM, CONVDIFF))
CORPUS = 97          # not a multiple of any lane width / tile: exercises tails
SEED = 20261018


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def refelem():
    out = {}
    for et in ElementType:
        rule, table = reference_element(et)
        out[f"{et.value}_points"] = rule.points
        out[f"{et.value}_weights"] = rule.weights
        out[f"{et.value}_values"] = table.values
        out[f"{et.value}_local_derivatives"] = table.local_derivatives
    _save("refelem.npz", **out)


def corpora():
    rng = np.random.default_rng(SEED)
    for element, problem in CASES:
        elements = [(random_geometry(element, rng), random_coefficients(problem, element, rng))
                    for _ in range(CORPUS)]
        batch = build_batch(elements)
        arrays = {
            "geometry_rows": batch.geometry_rows(),
            "coefficient_rows": batch.coefficient_rows(),
        }
        for desc in case_descriptors(element, problem):
            res = integrate_batch(desc, batch)
            arrays[f"A_{desc.short_name()}"] = res.stiffness
            arrays[f"b_{desc.short_name()}"] = res.load
        alg1 = [integrate_reference(g, c) for g, c in elements]
        arrays["A_algorithm1"] = np.stack([m.A for m in alg1])
        arrays["b_algorithm1"] = np.stack([m.b for m in alg1])
        _save(f"corpus_{element.value}_{problem.value}.npz", **arrays)


def twisted_prisms():
    """Acceptance case test_acceptance.py:132-166, with the refined-rule oracle."""
    rng = np.random.default_rng(SEED + 1)
    twist = 3e-6
    geo, cd_rows, po_rows, A_cd, b_cd, A_po, b_po = [], [], [], [], [], [], []
    for _ in range(12):
        ref = PRISM.reference_vertices.copy()
        ref[:, :2] += rng.uniform(-1.0, 1.0, size=(6, 2)) * twist
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        linear = q @ np.diag(rng.uniform(0.5, 2.0, size=3))
        g = ElementGeometry(PRISM, ref @ linear.T + rng.uniform(-1, 1, size=3))
        cd = random_coefficients(CONVDIFF, PRISM, rng)
        po = CoefficientSet.poisson(np.full(6, rng.uniform(0.5, 2.0)))
        geo.append(g.coords.reshape(-1))
        cd_rows.append(cd.flat())
        po_rows.append(po.flat())
        m = integrate_high_order(g, cd, level=4)
        A_cd.append(m.A)
        b_cd.append(m.b)
        m = integrate_high_order(g, po, level=4)
        A_po.append(m.A)
        b_po.append(m.b)
    _save("twisted_prisms.npz", geometry_rows=np.stack(geo), convdiff_rows=np.stack(cd_rows),
          poisson_rows=np.stack(po_rows), A_convdiff=np.stack(A_cd), b_convdiff=np.stack(b_cd),
          A_poisson=np.stack(A_po), b_poisson=np.stack(b_po))


def meshes():
    out = {}
    specs = {
        "tet_432": (MeshSpec(4, 3, 2, TET), 7, CONVDIFF),
        "tet_222": (MeshSpec(2, 2, 2, TET), 3, POISSON),
        "prism_53": (MeshSpec(5, 3, 1, PRISM), 11, CONVDIFF),
        "prism_44": (MeshSpec(4, 4, 1, PRISM), 0, POISSON),
    }
    for name, (spec, seed, problem) in specs.items():
        batch = generate_mesh(spec, seed, problem)
        out[f"{name}_geometry_rows"] = batch.geometry_rows()
        out[f"{name}_coefficient_rows"] = batch.coefficient_rows()
        out[f"{name}_spec"] = np.array([spec.nx, spec.ny, spec.nz, seed])
    _save("meshes.npz", **out)


def _error_of(desc, batch):
    try:
        integrate_batch(desc, batch)
    except GeometryError as err:
        kind = 1 if type(err).__name__ == "DegenerateElement" else 2
        point = -1 if err.point_index is None else err.point_index
        return np.array([kind, err.element_index, point]), str(err)
    raise AssertionError("expected a geometry error")


def block_rule_rows(good, partly, n=8300):
    """Shifted copies of the reference prism; 100 partly and 8200 fully inverted."""
    rows = np.tile(good.reshape(-1), (n, 1))
    rows[:, 0::3] += 1e-3 * np.arange(n)[:, None]
    rows[100] = partly.reshape(-1)
    rows[8200] = -good.reshape(-1)
    return rows


def error_cases():
    """First-error semantics, including the 8192-block and smallest-q rules."""
    rng = np.random.default_rng(SEED + 2)
    out, messages = {}, []

    def tet_batch(n, bad):
        els = [(random_geometry(TET, rng), random_coefficients(POISSON, TET, rng)) for _ in range(n)]
        for e, coords in bad.items():
            els[e] = (ElementGeometry(TET, coords), els[e][1])
        return build_batch(els)

    inverted = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, -1]], dtype=float)
    flat = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], dtype=float)
    cases = {
        "tet_inverted_4_7": (tet_batch(9, {4: inverted, 7: inverted}), TET, POISSON),
        "tet_degenerate_3_inverted_1": (tet_batch(6, {3: flat, 1: inverted}), TET, POISSON),
    }
    # prism that is fine at q < 3 but inverted at the top layer points:
    # pull the top face through the bottom face at one vertex
    good = PRISM.reference_vertices.copy()
    partly = good.copy()
    partly[5, 2] = -3.0   # vertex 5 (top, above vertex 2) drops below the bottom
    pr = [(random_geometry(PRISM, rng), random_coefficients(CONVDIFF, PRISM, rng)) for _ in range(20)]

    def prism_batch(n, bad):
        els = [(random_geometry(PRISM, rng), random_coefficients(CONVDIFF, PRISM, rng)) for _ in range(n)]
        for e, coords in bad.items():
            els[e] = (ElementGeometry(PRISM, coords), els[e][1])
        return build_batch(els)

    degenerate_prism = good.copy()
    degenerate_prism[3:] = degenerate_prism[:3]
    cases["prism_degenerate_2"] = (prism_batch(6, {2: degenerate_prism}), PRISM, CONVDIFF)
    cases["prism_partial_5_full_7"] = (prism_batch(12, {5: partly, 7: -good}), PRISM, CONVDIFF)
    # fails at q = 1..5 but not at q = 0: the reported point must be the
    # smallest failing q (1), not the first one a zeta-major traversal meets (2)
    min_q = np.array([[1.0735260056398386, 0.12576261533222466, -0.8115836684702022], [1.477080626165721, -1.160412031527824, -0.07387428460248158], [-0.12848346302867486, 0.18727422292154416, 0.00080667169439685], [-1.1216759257033364, 0.411796613002633, -0.23779211946897516], [0.7747694645679373, 0.767314309052276, 1.2606507785965007], [-0.7160999048204778, 0.18610641169245237, 2.4502436484894625]])
    cases["prism_min_q_3"] = (prism_batch(8, {3: min_q}), PRISM, CONVDIFF)
    # block rule: element 8200 fails at q=0 (block 1), element 100 only at a
    # later q (block 0).  Geometry is a formula (block_rule_rows) so the
    # fixture does not have to store 8300 elements.
    cases["prism_block_rule"] = (
        ElementBatch.from_arrays(PRISM, CONVDIFF, block_rule_rows(good, partly),
                                 np.zeros((8300, 20))), PRISM, CONVDIFF)
    del pr
    for name, (batch, element, problem) in cases.items():
        for desc in case_descriptors(element, problem):
            code, msg = _error_of(desc, batch)
            out[f"{name}__{desc.short_name()}"] = code
            messages.append(f"{name}__{desc.short_name()}\t{msg}")
        if name != "prism_block_rule":
            out[f"{name}__geometry_rows"] = batch.geometry_rows()
            out[f"{name}__coefficient_rows"] = batch.coefficient_rows()
    out["prism_partly_inverted"] = partly
    _save("errors.npz", **out)
    with open(os.path.join(HERE, "error_messages.tsv"), "w") as fh:
        fh.write("\n".join(messages) + "\n")


def unit_elements():
    """Analytic goldens of test_kernels.py:55-85 / test_acceptance.py:169-196."""
    out = {}
    for et in ElementType:
        geom = ElementGeometry(et, et.reference_vertices)
        for problem in ProblemClass:
            coeff = CoefficientSet.poisson(np.ones(et.n_quad)) if problem is POISSON else \
                CoefficientSet.convdiff(np.eye(4), np.ones(4))
            batch = build_batch([(geom, coeff)])
            for desc in case_descriptors(et, problem):
                res = integrate_batch(desc, batch)
                out[f"A_{desc.short_name()}"] = res.stiffness[0]
                out[f"b_{desc.short_name()}"] = res.load[0]
    _save("unit_elements.npz", **out)


SLICE = 1024  # sampled elements per benchmark configuration


def bench_slices(keys=("C1", "C2", "C3", "C4", "C5T", "C5P")):
    """The benchmark configurations end to end through the reference.

    The full mesh comes from the reference's own generate_mesh (coefficient
    seed as in the benchmark).  Prism configurations add the benchmark's
    top-face jitter, restated by paper_1504_01023_b200.mesh.jitter_top_faces,
    since the reference applies it only in its verification corpus
    (verify.py:85-86).  1024 sampled elements are then integrated by the
    reference's integrate_batch with the natural QSS descriptor: the first
    and last 128 elements plus 768 seeded random ones.  The GPU test
    regenerates each configuration with the device mesh generator, checks the
    sampled inputs bit for bit, and compares its outputs with the
    reference's.
    """
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1504_01023_b200 import mesh as M  # host restatement: specs and jitter only

    for key in keys:
        cfg = M.bench_configs()[key]
        spec = MeshSpec(cfg.spec.nx, cfg.spec.ny, cfg.spec.nz, ElementType(cfg.spec.element_type.value))
        problem = ProblemClass(cfg.problem.value)
        batch = generate_mesh(spec, cfg.coeff_seed, problem)
        geo, cof = batch.geometry_rows(), batch.coefficient_rows()
        if cfg.jitter_seed is not None:
            geo = M.jitter_top_faces(geo, cfg.spec, cfg.jitter_seed)
        n = geo.shape[0]
        rng = np.random.default_rng(SEED + 7)
        idx = np.unique(np.concatenate([np.arange(128), np.arange(n - 128, n),
                                        rng.choice(n, SLICE - 256, replace=False)]))
        g, c = np.ascontiguousarray(geo[idx]), np.ascontiguousarray(cof[idx])
        desc = case_descriptors(spec.element_type, problem)[0]
        res = integrate_batch(desc, ElementBatch.from_arrays(spec.element_type, problem, g, c))
        _save(f"bench_{key}.npz", index=idx, geometry_rows=g, coefficient_rows=c, A=res.stiffness, b=res.load,
              n_elements=np.array([n]))
        del batch, geo, cof


if __name__ == "__main__":
    print("reference feklab", feklab.__version__, "from", os.path.dirname(feklab.__file__), file=sys.stderr)
    if sys.argv[1:] == ["bench"]:
        bench_slices()
        sys.exit(0)
    refelem()
    corpora()
    twisted_prisms()
    meshes()
    error_cases()
    unit_elements()
    bench_slices()
