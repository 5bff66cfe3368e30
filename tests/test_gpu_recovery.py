"""Strain/stress recovery on the GPU (fsfem_recover_stress) vs oracle O9
(Eq. 2/4 evaluated literally) on the same displacements, plus a solved beam."""
import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam
from oracle import Oracle

pytestmark = pytest.mark.gpu

E, NU = 1.0e6, 0.3


@pytest.fixture(scope="module")
def fs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2001_08849_b200 import FsFem, load_library
    load_library()
    return FsFem


@pytest.mark.parametrize("name", ["ragged_perm", "cfg2"])
def test_recovery_matches_oracle_random_u(fs, name):
    m = (kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8, tet_perm_seed=9)
         if name == "ragged_perm" else config_mesh(2))
    u = np.random.default_rng(3).standard_normal(3 * m.n_nodes) * 1e-3
    g = fs()
    nf, _ = g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    eps, sig, ns, vm = g.recover_stress(u, nf)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    oeps, osig, ons, ovm = o.recover(E, NU, u)
    for a, b in ((eps, oeps), (sig, osig), (ns, ons), (vm, ovm)):
        assert np.abs(a - b).max() <= 1e-10 * np.abs(b).max()


def test_recovery_of_solved_beam(fs):
    """cfg2 solved on the GPU: max von Mises at the clamped end (Fig. 13's qualitative
    check), and the GPU recovery of that solution equals the oracle's."""
    m = config_mesh(2)
    g = fs()
    nf, _ = g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve()
    eps, sig, ns, vm = g.recover_stress(u, nf)
    x = m.xyz[:, 0]
    assert x[np.argmax(vm)] <= 0.1 * x.max()
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    _, _, ons, ovm = o.recover(E, NU, u)
    assert np.abs(vm - ovm).max() <= 1e-10 * ovm.max()


def test_recovery_fem_t4_linear_field(fs):
    """FEM-T4 domains are the tets: a linear field gives its exact constant strain in every tet."""
    from paper_2001_08849_b200 import METHOD_FEM_T4
    m = kuhn_beam(4, 3, 2, L=2.0, jitter=0.2, jitter_seed=7)
    G = np.random.default_rng(1).standard_normal((3, 3)) * 1e-3
    u = (m.xyz @ G.T).reshape(-1)
    g = fs()
    g.set_method(METHOD_FEM_T4)
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    eps, sig, ns, vm = g.recover_stress(u, m.n_tets)
    ref = np.array([G[0, 0], G[1, 1], G[2, 2], G[1, 2] + G[2, 1], G[0, 2] + G[2, 0], G[0, 1] + G[1, 0]])
    assert np.abs(eps - ref).max() <= 1e-10 * np.abs(ref).max()
