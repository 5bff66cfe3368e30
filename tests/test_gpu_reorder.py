"""Internal node renumbering (fsfem_set_reorder): with the nodes stored in Morton
order inside the library, every output in the caller's numbering must equal the oracle's exactly
as without renumbering (faces and CSR pattern bit-exact, values 1e-12, u 1e-7)."""
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


MESHES = {"cfg2": lambda: config_mesh(2),
          "ragged_perm": lambda: kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8,
                                           tet_perm_seed=9)}


@pytest.mark.parametrize("name", list(MESHES))
def test_reordered_path_matches_oracle(fs, name):
    m = MESHES[name]()
    g = fs()
    g.set_reorder(1)
    g.build_faces(m.xyz, m.tets)
    assert g.report()["reordered"] == 1
    o = Oracle(m.xyz, m.tets)
    ofn, oft, ofo = o.build_faces()
    fn, ft, fo = g.get_faces()
    assert np.array_equal(fn, ofn) and np.array_equal(ft, oft) and np.array_equal(fo, ofo)
    g.assemble_csr(E, NU)
    c = g.get_csr()
    _, orp, oci, ova = o.assemble_fs(E, NU)
    kmax = np.abs(ova).max()
    assert np.array_equal(c.row_ptr, orp) and np.array_equal(c.col_idx, oci)
    assert np.abs(c.vals - ova).max() <= 1e-12 * kmax
    x = np.random.default_rng(2).standard_normal(3 * m.n_nodes)
    assert np.abs(g.spmv(x) - o.spmv(x)).max() <= 1e-11 * kmax * np.abs(x).max()
    top = np.isclose(m.xyz[:, 2], m.xyz[:, 2].max())
    assert np.abs(g.surface_loads(top, [0.0, 0.0, -1.0]) - o.surface_loads(top, [0.0, 0.0, -1.0])).max() <= 1e-14
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    orp2, oci2, ova2, _ = o.apply_bc(m.dirichlet, m.loads, 0)
    c2 = g.get_csr()
    assert np.abs(c2.vals - ova2).max() <= 1e-12 * kmax
    u, rep = g.pcg_solve()
    uo, _ = o.pcg(1e-10)
    assert rep["converged"] == 1
    assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)
    eps, sig, ns, vm = g.recover_stress(u, g.n_faces)
    _, _, ons, ovm = o.recover(E, NU, u)
    assert np.abs(vm - ovm).max() <= 1e-10 * ovm.max()
    assert np.abs(ns - ons).max() <= 1e-10 * np.abs(ons).max()


def test_auto_reorder_triggers_on_random_numbering(fs):
    """cfg3 with its nodes randomly relabelled (like cfg5): auto mode renumbers, the natural
    numbering does not, and both give the same displacements in the caller's numbering."""
    base = config_mesh(3)
    perm = kuhn_beam(100, 20, 20, L=10.0, jitter=0.15, jitter_seed=3, node_perm_seed=77, tet_perm_seed=78)
    out = {}
    for key, m in (("natural", base), ("perm", perm)):
        g = fs()
        g.build_faces(m.xyz, m.tets)
        reordered = g.report()["reordered"]
        g.assemble_csr(E, NU)
        g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        u, rep = g.pcg_solve()
        out[key] = (reordered, m, u)
    assert out["natural"][0] == 0 and out["perm"][0] == 1
    # same beam: compare tip deflections (the two meshes are the same geometry and loads)
    tips = [u.reshape(-1, 3)[m.tip, 2].mean() for _, m, u in out.values()]
    assert abs(tips[0] - tips[1]) <= 1e-7 * abs(tips[0])


def test_reordered_solve_is_bitwise_reproducible(fs):
    """The internal Morton order (device radix sort, ties by node id) and everything after it are
    pure functions of the input: two full runs on a randomly relabelled mesh give identical bytes."""
    m = kuhn_beam(24, 6, 6, L=4.0, jitter=0.2, jitter_seed=3, node_perm_seed=5, tet_perm_seed=6)
    outs = []
    for _ in range(2):
        g = fs()
        g.set_reorder(1)
        g.build_faces(m.xyz, m.tets)
        g.assemble_csr(E, NU)
        v = g.get_csr(with_pattern=False).vals.copy()
        g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        u, rep = g.pcg_solve()
        assert rep["reordered"] == 1
        outs.append((v, u, rep["iterations"]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1]) and outs[0][2] == outs[1][2]
