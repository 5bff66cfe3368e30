"""The paper's own validation case (§4.1; Table 4 at 590-603; SURVEY.md 8(f)
f4) on a locally generated mesh: a 1 x 0.2 x 0.2 m cantilever, E = 2e8, nu = 0.3, clamped at
x = 0 with the penalty method, uniform pressure p = 12,500 N/m^2 on the upper
face in -z turned into nodal loads p*A/3 (fsfem_surface_loads).  The paper's TetGen mesh (458
nodes, 1,576 T4) is not available; a Kuhn mesh of 20x4x4 hexes (525 nodes, 1,920 T4) stands in,
so Table 4 is matched only loosely, while the ordering FEM-T4 < FS-FEM < T10 and the parity with
the oracle are exact checks."""
import numpy as np
import pytest

from fsfem_inputs import kuhn_beam
from oracle import Oracle

pytestmark = pytest.mark.gpu

E, NU, P = 2.0e8, 0.3, 12500.0
L, W, H = 1.0, 0.2, 0.2
TABLE4_X = [0.2, 0.4, 0.6, 0.8, 1.0]
TABLE4 = {"fem": [-8.20e-4, -2.61e-3, -4.99e-3, -7.62e-3, -1.03e-2],   # FEM-T4 column
          "fs": [-8.66e-4, -2.82e-3, -5.41e-3, -8.28e-3, -1.12e-2],    # juSFEM-T4 column
          "t10": [-9.54e-4, -3.08e-3, -5.86e-3, -8.92e-3, -1.20e-2]}   # ABAQUS FEM-T10 column


@pytest.fixture(scope="module")
def fs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2001_08849_b200 import FsFem, load_library
    load_library()
    return FsFem


def _mesh():
    m = kuhn_beam(20, 4, 4, L=L, W=W, H=H)
    return m, np.isclose(m.xyz[:, 2], H), np.nonzero(np.isclose(m.xyz[:, 0], 0.0))[0].astype(np.int32)


def _solve(fs, method):
    from paper_2001_08849_b200 import METHOD_FEM_T4, METHOD_FS
    m, top, clamped = _mesh()
    g = fs()
    g.set_method(METHOD_FEM_T4 if method == "fem" else METHOD_FS)
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    loads = g.surface_loads(top, [0.0, 0.0, -P])
    g.apply_bc(clamped, loads.reshape(-1), 1)  # PENALTY
    u, rep = g.pcg_solve(rel_tol=1e-10)
    assert rep["converged"] == 1
    return m, loads, u


def _deflection_curve(m, u):
    uz = u.reshape(-1, 3)[:, 2]
    return np.array([uz[np.isclose(m.xyz[:, 0], x)].mean() for x in TABLE4_X])


def test_pressure_loads_match_oracle(fs):
    m, top, clamped = _mesh()
    g = fs()
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    loads = g.surface_loads(top, [0.0, 0.0, -P])
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    ref = o.surface_loads(top, [0.0, 0.0, -P])
    assert np.abs(loads - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.isclose(loads[:, 2].sum(), -P * L * W, rtol=1e-12)


def test_paper_41_cantilever(fs):
    m, loads, u_fs = _solve(fs, "fs")
    _, _, u_fem = _solve(fs, "fem")
    d_fs, d_fem = _deflection_curve(m, u_fs), _deflection_curve(m, u_fem)
    # oracle parity of the FS solve (same loads, PENALTY)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    o.assemble_fs(E, NU)
    o.apply_bc(np.nonzero(np.isclose(m.xyz[:, 0], 0.0))[0].astype(np.int32), loads, 1)
    uo, _ = o.pcg(1e-10)
    assert np.linalg.norm(u_fs - uo) <= 1e-6 * np.linalg.norm(uo)
    # ordering of Table 4 at every station: |FEM-T4| < |FS-FEM| < |T10|
    assert np.all(np.abs(d_fem) < np.abs(d_fs)) and np.all(np.abs(d_fs) < np.abs(TABLE4["t10"]))
    # loose agreement with the paper's juSFEM-T4 / FEM-T4 columns (different mesh family)
    assert np.all(np.abs(d_fs - TABLE4["fs"]) <= 0.15 * np.abs(TABLE4["fs"])), d_fs
    assert np.all(np.abs(d_fem - TABLE4["fem"]) <= 0.15 * np.abs(TABLE4["fem"])), d_fem
