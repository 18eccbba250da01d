"""Device mesh generation (fek_mesh_geometry / fek_pcg64_uniform) is bit-identical to the host generator."""

import numpy as np
import pytest

from paper_1504_01023_b200 import ElementType, ProblemClass, mesh

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec,jitter", [
    (mesh.MeshSpec(7, 5, 3, ElementType.TETRAHEDRON), None),
    (mesh.MeshSpec(31, 17, 1, ElementType.PRISM), None),
    (mesh.MeshSpec(31, 17, 1, ElementType.PRISM), 3),
])
def test_geometry_bitwise(spec, jitter):
    host = mesh.geometry_rows(spec)
    if jitter is not None:
        host = mesh.jitter_top_faces(host, spec, jitter)
    dev = mesh.device_geometry(spec, jitter_seed=jitter).cpu().numpy().reshape(host.shape)
    assert np.array_equal(dev, host)
    rng = np.random.default_rng(0)
    for _ in range(5):
        lo = int(rng.integers(0, spec.n_elements))
        hi = int(rng.integers(lo, spec.n_elements + 1))
        part = mesh.device_geometry(spec, lo, hi - lo, jitter).cpu().numpy().reshape(-1, host.shape[1])
        assert np.array_equal(part, host[lo:hi])


@pytest.mark.parametrize("problem,etype,seed", [(ProblemClass.CONV_DIFF, ElementType.TETRAHEDRON, 0),
                                                (ProblemClass.POISSON, ElementType.PRISM, 7)])
def test_coefficients_bitwise(problem, etype, seed):
    n = 10007
    host = mesh.coefficient_rows(n, problem, etype, seed)
    dev = mesh.device_coefficients(problem, etype, seed, 0, n).cpu().numpy().reshape(host.shape)
    assert np.array_equal(dev, host)
    part = mesh.device_coefficients(problem, etype, seed, 4321, 999).cpu().numpy().reshape(-1, host.shape[1])
    assert np.array_equal(part, host[4321:5320])


def test_config_slices_match_host_at_scale():
    cfg = mesh.bench_configs()["C3"]
    geo_h, cof_h = mesh.config_rows(cfg)
    lo, n = 1_234_567, 100_000
    g, c = mesh.device_config(cfg, lo, n)
    assert np.array_equal(g.cpu().numpy().reshape(n, -1), geo_h[lo:lo + n])
    assert np.array_equal(c.cpu().numpy().reshape(n, -1), cof_h[lo:lo + n])
