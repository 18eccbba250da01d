"""GPU halves of the CLI / bench / verify mirror (``pkg/tests/test_bench_cli.py``).

``verify`` checks every descriptor's CUDA results against the naive checker;
``bench`` / ``tune`` time the kernels after the gate and emit the reference's
CSV schema; geometry failures exit 3, gate failures 1.
"""

import numpy as np
import pytest

from conftest import golden
from paper_1504_01023_b200 import (BUILTIN_PROFILES, DeviceBatch, ElementGeometry, ElementType, GeometryPath,
                                   KernelDescriptor, ProblemClass, Variant, build_batch, read_batch, write_batch)
from paper_1504_01023_b200.bench import CSV_COLUMNS, run_benchmark
from paper_1504_01023_b200.cli import main
from paper_1504_01023_b200.mesh import MeshSpec, generate_mesh
from paper_1504_01023_b200.verify import random_coefficients, random_geometry, run_verification

pytestmark = [pytest.mark.gpu, pytest.mark.filterwarnings("ignore:per-run time below")]

TET = ElementType.TETRAHEDRON
DESC = KernelDescriptor(Variant.QSS, GeometryPath.GEO_LINEAR, ProblemClass.POISSON, TET)


def test_run_verification_all_descriptors():
    report = run_verification(per_case=40, seed=5)
    assert report.passed, report.summary_lines()
    assert len(report.cases) == 4
    assert report.max_rel_err < 1e-13


def test_run_verification_strict_tolerance_fails():
    report = run_verification(per_case=3, seed=1, tolerance=1e-18)
    assert not report.passed
    assert any("rel err" in line for line in report.summary_lines())


def test_run_benchmark_record_device_and_host():
    batch = generate_mesh(MeshSpec(8, 8, 8, TET), 3, ProblemClass.POISSON)
    for inputs in ("device", "host"):
        rec = run_benchmark(batch, DESC, BUILTIN_PROFILES["xeon-e5"], repeats=3, inputs=inputs)
        assert rec.ns_per_element > 0 and rec.measured_accesses == 36
        assert rec.model_bound_ns == pytest.approx(4.2985, abs=0.001)
        assert rec.worker_count == 1 and rec.n_elements == 3072
    dev = DeviceBatch.from_host(generate_mesh(MeshSpec(64, 64, 64, TET), 3, ProblemClass.POISSON))
    rec = run_benchmark(dev, DESC, BUILTIN_PROFILES["k20m"], repeats=3)
    assert rec.efficiency_pct > 100       # 1.57M resident tets: a B200 beats the K20m bound by far


def test_cli_verify_ok(capsys):
    assert main(["verify", "--elements", "10", "--seed", "5"]) == 0
    assert "PASSED" in capsys.readouterr().out


def test_cli_genmesh_and_bench_roundtrip(tmp_path):
    mesh = tmp_path / "mesh.fekb"
    assert main(["genmesh", "--element", "prism", "--problem", "convdiff", "--elements", "5000",
                 "--out", str(mesh)]) == 0
    for inputs in ("device", "host"):
        out = tmp_path / f"runs_{inputs}.csv"
        assert main(["bench", "--element", "prism", "--problem", "convdiff", "--batch", str(mesh), "--repeats", "3",
                     "--format", "csv", "--out", str(out), "--inputs", inputs]) == 0
        lines = out.read_text().strip().split("\n")
        assert lines[0] == ",".join(CSV_COLUMNS) and len(lines) == 2
        row = dict(zip(CSV_COLUMNS, lines[1].split(",")))
        assert row["accesses_per_element"] == "80" and row["n_elements"] == str(read_batch(mesh).n_elements)


def test_cli_bench_no_verify_marks_output(tmp_path, capsys):
    out = tmp_path / "runs.csv"
    assert main(["bench", "--elements", "50", "--repeats", "3", "--no-verify", "--format", "csv",
                 "--out", str(out)]) == 0
    assert out.read_text().startswith("# UNVERIFIED")
    assert "UNVERIFIED" in capsys.readouterr().err


def test_cli_tune_small(tmp_path):
    out = tmp_path / "tune.csv"
    assert main(["tune", "--elements", "64", "--repeats", "3", "--format", "csv", "--out", str(out),
                 "--workers", "2"]) == 0
    lines = out.read_text().strip().split("\n")
    assert lines[0] == ",".join(CSV_COLUMNS)
    assert len(lines) == 1 + 6 * 2


def test_cli_degenerate_mesh_exits_3(tmp_path, rng):
    elements = [(random_geometry(TET, rng), random_coefficients(ProblemClass.POISSON, TET, rng)) for _ in range(8)]
    coords = elements[3][0].coords.copy()
    coords[3] = coords[0]
    elements[3] = (ElementGeometry(TET, coords), elements[3][1])
    path = tmp_path / "bad.fekb"
    write_batch(build_batch(elements, pad_value=0.0), path)
    assert main(["bench", "--batch", str(path), "--repeats", "3", "--no-verify"]) == 3
    assert main(["bench", "--batch", str(path), "--repeats", "3", "--no-verify", "--inputs", "host"]) == 3


def test_cli_bench_gate_failure_exits_1(monkeypatch, capsys):
    import paper_1504_01023_b200.cli as cli

    class Failing:
        passed = False
        tolerance = 1e-12
        max_rel_err = 1.0

        @staticmethod
        def summary_lines():
            return ["injected failure"]

    monkeypatch.setattr(cli, "run_verification", lambda **kw: Failing())
    assert main(["bench", "--elements", "50", "--repeats", "3"]) == 1
    assert "injected failure" in capsys.readouterr().err


def test_verify_batch_results_match_reference_corpus():
    """The gate's batch leg on the reference corpus reproduces the reference's own batch output."""
    from paper_1504_01023_b200 import ElementBatch, integrate_batch
    from paper_1504_01023_b200.problems import case_descriptors
    from paper_1504_01023_b200.verify import relative_difference

    for et, pb in ((TET, ProblemClass.CONV_DIFF), (ElementType.PRISM, ProblemClass.CONV_DIFF)):
        g = golden(f"corpus_{et.value}_{pb.value}.npz")
        batch = ElementBatch.from_arrays(et, pb, g["geometry_rows"], g["coefficient_rows"])
        for desc in case_descriptors(et, pb):
            res = integrate_batch(desc, batch)
            assert relative_difference(res.stiffness, g[f"A_{desc.short_name()}"]) <= 1e-12
            assert np.isfinite(res.load).all()


def test_extended_tuner_sweeps_tiles_and_ctas(tmp_path):
    """tune --launch: tile T x CTAs/SM rows in the reference's CSV schema plus two trailing columns."""
    import csv

    from paper_1504_01023_b200 import tune

    out = tmp_path / "launch.csv"
    assert tune.main(["--case", "C3", "--elements", "40000", "--repeats", "2", "--launch", "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert {int(r["tile_elements"]) for r in rows} == {64, 128, 256}
    assert min(int(r["ctas_per_sm"]) for r in rows) == 1 and len(rows) >= 4
    assert list(rows[0].keys())[-2:] == ["tile_elements", "ctas_per_sm"]
    assert all(float(r["ns_per_element"]) > 0 for r in rows)
