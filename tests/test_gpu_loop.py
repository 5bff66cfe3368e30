"""PCG loop control: the default device-side loop (one CUDA-graph launch
whose while node repeats the iteration body until the device-side recurrence stops, no host
synchronisation inside the solve) gives bitwise the same solve as host-polled graph batches, and
every PCG SpMV launch is timed on the device."""
import numpy as np
import pytest

from fsfem_inputs import config_mesh

pytestmark = pytest.mark.gpu

E, NU = 1.0e6, 0.3


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2001_08849_b200 as P
    P.load_library()
    return P


@pytest.mark.parametrize("cfg,variant", [(1, 0), (2, 0), (2, 1), (3, 0)])
def test_device_loop_equals_host_loop(P, cfg, variant):
    m = config_mesh(cfg)
    out = {}
    for mode in (1, 0):
        g = P.FsFem()
        g.set_loop(mode)
        g.set_pcg_variant(variant)
        g.build_faces(m.xyz, m.tets)
        g.assemble_csr(E, NU)
        g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        u, rep = g.pcg_solve(rel_tol=1e-10)
        out[mode] = (u, rep)
        g.close()
    (uh, rh), (ud, rd) = out[1], out[0]
    assert rd["converged"] == 1 and rd["iterations"] == rh["iterations"]
    assert np.array_equal(ud, uh)
    if variant == 0:  # one SpMV per iteration, each timed on the device
        assert rd["spmv_launches"] == rd["iterations"]
        assert rd["t_spmv_ms"] > 0.0


def test_loop_mode_errors(P):
    g = P.FsFem()
    with pytest.raises(P.FsfemError) as e:
        g.set_loop(7)
    assert e.value.status == "INVALID_ARG"
    g.close()
