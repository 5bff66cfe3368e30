"""FEM-T4 on the GPU: the conventional linear-tet stiffness through the same
C ABI (fsfem_set_method), against the oracle's FEM-T4 (oracle O8), and the
theorem FS-FEM tip deflection >= FEM-T4 (K_FS <= K_FEM in the Loewner order)."""
import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam, kuhn_counts
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


def _gpu(fs, m, method):
    from paper_2001_08849_b200 import METHOD_FEM_T4, METHOD_FS
    g = fs()
    g.set_method(METHOD_FEM_T4 if method == "fem" else METHOD_FS)
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    return g


MESHES = {"cfg1": lambda: config_mesh(1), "cfg2": lambda: config_mesh(2),
          "ragged_perm": lambda: kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8,
                                           tet_perm_seed=9)}


@pytest.mark.parametrize("name", list(MESHES))
def test_fem_csr_parity(fs, name):
    m = MESHES[name]()
    g = _gpu(fs, m, "fem")
    c = g.get_csr()
    o = Oracle(m.xyz, m.tets)
    _, orp, oci, ova = o.assemble_fem(E, NU)
    assert np.array_equal(c.row_ptr, orp) and np.array_equal(c.col_idx, oci)
    assert np.abs(c.vals - ova).max() <= 1e-12 * np.abs(ova).max()
    if name.startswith("cfg"):
        assert g.nnz == kuhn_counts(*m.grid)["nnz_fem"]


@pytest.mark.parametrize("name", ["cfg1", "ragged_perm"])
def test_fem_solve_parity(fs, name):
    m = MESHES[name]()
    g = _gpu(fs, m, "fem")
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve(rel_tol=1e-10)
    o = Oracle(m.xyz, m.tets)
    o.assemble_fem(E, NU)
    o.apply_bc(m.dirichlet, m.loads, 0)
    uo, _ = o.pcg(1e-10)
    assert rep["converged"] == 1
    assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)


def test_single_tet_fs_equals_fem(fs):
    """One tet: 4 exterior faces, each a quarter of the tet with B = the tet's B -> K_FS = K_FEM."""
    xyz = np.array([[0, 0, 0], [1.0, 0.1, 0], [0.2, 1.1, 0.1], [0.3, 0.2, 0.9]])
    tets = np.array([[0, 1, 2, 3]], np.int32)
    m = type("M", (), {"xyz": xyz, "tets": tets})
    a = _gpu(fs, m, "fs").get_csr()
    b = _gpu(fs, m, "fem").get_csr()
    assert np.array_equal(a.col_idx, b.col_idx)
    assert np.abs(a.vals - b.vals).max() <= 1e-12 * np.abs(b.vals).max()


@pytest.mark.parametrize("cfg", [3, 4])
def test_fs_deflects_more_than_fem(fs, cfg):
    """Tip compliance f.u: FS-FEM >= FEM-T4 (theorem), both from the GPU."""
    m = config_mesh(cfg)
    f = m.loads.reshape(-1)
    out = {}
    for method in ("fs", "fem"):
        g = _gpu(fs, m, method)
        g.apply_bc(m.dirichlet, f)
        u, rep = g.pcg_solve(rel_tol=1e-10)
        assert rep["converged"] == 1
        out[method] = f @ u
    assert out["fs"] >= out["fem"] > 0


def test_method_switch_rebuilds(fs):
    from paper_2001_08849_b200 import METHOD_FEM_T4, METHOD_FS
    m = MESHES["cfg1"]()
    g = fs()
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    nnz_fs = g.nnz
    g.set_method(METHOD_FEM_T4)
    g.assemble_csr(E, NU)
    assert g.nnz == kuhn_counts(*m.grid)["nnz_fem"] < nnz_fs
    g.set_method(METHOD_FS)
    g.assemble_csr(E, NU)
    assert g.nnz == nnz_fs
