"""Full-size parity at the BASELINE.json configurations (GPU).

Every element of C1 (1.05M tets, Poisson), C3 (4.0M jittered prisms, Poisson)
and C4 (16.0M jittered prisms, CDR) is integrated on the GPU and compared with
the CPU oracle (bitwise-pinned numpy restatement of the reference, run on all
host cores): max relative Frobenius error <= 1e-12 for A and b.  C2 is covered
the same way by bench.py's parity record.

Also at full size: the fek_checksum bit-pattern sums of a single launch equal
the sum over 8 contiguous sharded launches (base_index offsets) bit for bit --
the multi-GPU independence property, exercised on one GPU.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", ["C1", "C3", "C4"])
def test_full_config_parity(key):
    import torch

    from oracle import numpy_oracle as O
    from oracle.cpu_baseline import PortPool
    from paper_1504_01023_b200 import ELEMENT_MAJOR, DeviceBatch, KernelDescriptor, integrate_batch, mesh, natural_path
    from paper_1504_01023_b200.distributed import all_shards, device_checksum
    from paper_1504_01023_b200.problems import Variant

    cfg = mesh.bench_configs()[key]
    et, pb = cfg.spec.element_type, cfg.problem
    desc = KernelDescriptor(Variant.QSS, natural_path(et), pb, et)
    geo, cof = mesh.config_rows(cfg)
    n = geo.shape[0]
    dev = DeviceBatch(et, pb, n, ELEMENT_MAJOR, torch.from_numpy(geo.reshape(-1)).cuda(),
                      torch.from_numpy(cof.reshape(-1)).cuda())
    res = integrate_batch(desc, dev)
    f_all, u_all = device_checksum(res)

    # sharded launches: same bits
    u_sum = torch.zeros(2, dtype=torch.int64, device="cuda")
    for lo, hi in all_shards(n, 8):
        sub = DeviceBatch(et, pb, hi - lo, dev.layout, dev.geometry_data[lo * et.geometry_size: hi * et.geometry_size],
                          dev.coefficient_data[lo * cof.shape[1]: hi * cof.shape[1]])
        part = integrate_batch(desc, sub, base_index=lo)
        assert torch.equal(part.stiffness, res.stiffness[lo:hi])
        _, u = device_checksum(part, base_index=lo)
        u_sum += u
    assert torch.equal(u_sum, u_all)

    A_gpu = res.stiffness.cpu().numpy()
    b_gpu = res.load.cpu().numpy()
    del res, dev
    torch.cuda.empty_cache()
    with PortPool("qss", desc.geometry_path.value, pb.value, et.value, geo, cof) as pool:
        pool.run(0, n)
        errA = O.rel_frobenius(A_gpu, pool.A)
        errb = O.rel_frobenius(b_gpu, pool.b)
    print(f"{key}: {n} elements, max rel err A {errA.max():.3e} b {errb.max():.3e}, "
          f"median A {np.median(errA):.3e}")
    assert errA.max() <= 1e-12 and errb.max() <= 1e-12
