"""Benchmark configurations end to end against the REFERENCE (no oracle in between).

tests/golden/bench_<cfg>.npz holds, for each benchmark configuration, 1024
sampled elements of the full mesh as the reference's generate_mesh made it
(prisms with the benchmark's top-face jitter), and the reference's own
integrate_batch outputs for them (tests/golden/make_golden.py bench_slices).
Here the whole configuration is generated in HBM by the device mesh
generator and integrated in one launch.  The sampled inputs must match the
reference's bit for bit, and the outputs must agree to 1e-12.
"""

import numpy as np
import pytest

from conftest import golden
from paper_1504_01023_b200 import DeviceBatch, ELEMENT_MAJOR, case_descriptors, integrate_batch, mesh

pytestmark = pytest.mark.gpu


def rel_frobenius(got, want):
    axes = tuple(range(1, got.ndim))
    den = np.sqrt((want ** 2).sum(axis=axes))
    num = np.sqrt(((got - want) ** 2).sum(axis=axes))
    return np.where(den > 0, num / np.where(den > 0, den, 1.0), num)


@pytest.mark.parametrize("key", ["C1", "C2", "C3", "C4", "C5T", "C5P"])
def test_benchmark_configuration_matches_reference(key):
    import torch

    z = golden(f"bench_{key}.npz")
    cfg = mesh.bench_configs()[key]
    et, pb = cfg.spec.element_type, cfg.problem
    n = cfg.spec.n_elements
    assert int(z["n_elements"][0]) == n
    geo, cof = mesh.device_config(cfg)
    idx = torch.from_numpy(z["index"]).cuda()
    dsg, dsc = et.geometry_size, pb.coefficient_size(et)
    assert np.array_equal(geo.view(n, dsg).index_select(0, idx).cpu().numpy(), z["geometry_rows"])
    assert np.array_equal(cof.view(n, dsc).index_select(0, idx).cpu().numpy(), z["coefficient_rows"])
    res = integrate_batch(case_descriptors(et, pb)[0], DeviceBatch(et, pb, n, ELEMENT_MAJOR, geo, cof))
    A = res.stiffness.index_select(0, idx).cpu().numpy()
    b = res.load.index_select(0, idx).cpu().numpy()
    err = max(rel_frobenius(A, z["A"]).max(), rel_frobenius(b, z["b"]).max())
    print(f"{key}: {n} elements, sampled max rel Frobenius vs reference {err:.2e}")
    assert err <= 1e-12, err
    del res, geo, cof
    torch.cuda.empty_cache()
