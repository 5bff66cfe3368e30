"""Pins of the oracle's per-domain dense stiffness (ora_face_stiffness /
ora_tet_stiffness), each fixed by the paper or the mathematics rather than by the oracle's code:
  - FEM-T4 reference tet: entries written out by hand from grad N of the unit tet (V = 1/6) and
    sigma = lam tr(eps) I + 2 mu eps (textbook isotropic elasticity);
  - one-tet mesh: every (exterior) face has b = grad N and V_f = V_e / 4 (PAPER.md:128-136,
    Fig. 1: the cone of the face), so K_f = K_e / 4 in the face's field order;
  - two-tet interior face: u^T K_f u = V_f eps_bar : sigma(eps_bar) for random u, eps_bar the
    volume-weighted mean of the two tets' textbook strains (Eq. 7 smoothing);
  - any face or tet of a jittered mesh: symmetric, positive semi-definite, rank 6, the six rigid
    body modes in the null space (Eq. 9: V B^T c B with c of rank 6 and B annihilating rigid motions);
  - summed over the faces and scattered by field node, the K_f reproduce the oracle's assembled
    K (Eq. 12).
"""
import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam
from oracle import Oracle

E, NU = 2.0e8, 0.27
LAM = E * NU / ((1 + NU) * (1 - 2 * NU))
MU = E / (2 * (1 + NU))


def test_reference_tet_entries_by_hand():
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    o = Oracle(xyz, np.array([[0, 1, 2, 3]], np.int32))
    K, field = o.domain_stiffness(0, E, NU, tet=True)
    assert list(field) == [0, 1, 2, 3, -1]
    V = 1.0 / 6.0
    x, y, z = 0, 1, 2
    r = lambda node, comp: 3 * node + comp  # noqa: E731
    hand = {
        (r(1, x), r(1, x)): V * (LAM + 2 * MU),   # grad N1 = (1, 0, 0)
        (r(1, y), r(1, y)): V * MU,
        (r(1, x), r(1, y)): 0.0,
        (r(1, x), r(2, y)): V * LAM,              # grad N2 = (0, 1, 0)
        (r(1, y), r(2, x)): V * MU,
        (r(0, x), r(0, x)): V * (LAM + 4 * MU),   # grad N0 = (-1, -1, -1)
        (r(0, x), r(0, y)): V * (LAM + MU),
        (r(0, x), r(1, x)): -V * (LAM + 2 * MU),
        (r(0, y), r(1, x)): -V * LAM,
        (r(0, x), r(1, y)): -V * MU,
        (r(3, z), r(3, z)): V * (LAM + 2 * MU),
    }
    for (i, j), v in hand.items():
        assert abs(K[i, j] - v) <= 1e-12 * (LAM + 4 * MU), (i, j, K[i, j], v)
    assert np.all(K[12:, :] == 0) and np.all(K[:, 12:] == 0)


def _tet_grad(X):
    """Textbook gradients of the 4 linear shape functions: rows of inv([[1, x, y, z]])[1:].T."""
    A = np.hstack([np.ones((4, 1)), X])
    return np.linalg.inv(A)[1:].T  # [4 nodes, 3]


def test_single_tet_faces_are_quarter_of_element():
    rng = np.random.default_rng(3)
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float) + rng.uniform(-0.2, 0.2, (4, 3))
    tets = np.array([[0, 1, 2, 3]], np.int32)
    o = Oracle(xyz, tets)
    fn, ft, fo = o.build_faces()
    assert len(fn) == 4 and np.all(ft[:, 1] == -1)
    Ke, _ = o.domain_stiffness(0, E, NU, tet=True)
    for f in range(4):
        Kf, field = o.domain_stiffness(f, E, NU)
        assert field[4] == -1 and sorted(field[:4]) == [0, 1, 2, 3]
        idx = np.concatenate([3 * field[:4, None] + np.arange(3)]).ravel()  # tet order == node id here
        expect = Ke[np.ix_(idx, idx)] / 4.0
        assert np.abs(Kf[:12, :12] - expect).max() <= 1e-12 * np.abs(Ke).max(), f
        assert np.all(Kf[12:, :] == 0) and np.all(Kf[:, 12:] == 0)


def _strain(G):
    return 0.5 * (G + G.T)


def _energy_density(eps):
    sig = LAM * np.trace(eps) * np.eye(3) + 2 * MU * eps
    return np.sum(eps * sig)


def test_interior_face_energy_identity():
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.2, 0.3, 1.0], [0.3, 0.2, -2.1]], float)
    tets = np.array([[0, 1, 2, 3], [0, 1, 2, 4]], np.int32)
    o = Oracle(xyz, tets)
    fn, ft, fo = o.build_faces()
    f = int(np.flatnonzero(ft[:, 1] >= 0)[0])
    Kf, field = o.domain_stiffness(f, E, NU)
    assert list(field[:3]) == [0, 1, 2] and sorted(field[3:]) == [3, 4]
    V = [abs(np.linalg.det(xyz[t[1:]] - xyz[t[0]])) / 6.0 for t in tets]
    Vf = (V[0] + V[1]) / 4.0
    rng = np.random.default_rng(5)
    for _ in range(4):
        u = rng.standard_normal((5, 3))
        G = [(_tet_grad(xyz[t]).T @ u[t]).T for t in tets]  # G[i][a, b] = du_a / dx_b
        eps_bar = (V[0] * _strain(G[0]) + V[1] * _strain(G[1])) / (V[0] + V[1])
        uf = u[field].reshape(-1)
        lhs = uf @ Kf @ uf
        rhs = Vf * _energy_density(eps_bar)
        assert abs(lhs - rhs) <= 1e-11 * abs(rhs), (lhs, rhs)


def _rigid_modes(X):
    n = len(X)
    R = np.zeros((3 * n, 6))
    for i, (x, y, z) in enumerate(X):
        R[3 * i:3 * i + 3, :3] = np.eye(3)
        R[3 * i:3 * i + 3, 3:] = [[0, z, -y], [-z, 0, x], [y, -x, 0]]
    return R


@pytest.mark.parametrize("tet", [False, True])
def test_symmetric_psd_rank6_rigid_null(tet):
    m = config_mesh(1)
    o = Oracle(m.xyz, m.tets)
    fn, ft, fo = o.build_faces()
    n = len(m.tets) if tet else len(fn)
    ids = np.random.default_rng(9).choice(n, 24, replace=False)
    if not tet:
        ids = np.concatenate([ids, np.flatnonzero(ft[:, 1] < 0)[:4]])
    for k in ids:
        K, field = o.domain_stiffness(int(k), E, NU, tet=tet)
        nf = int((field >= 0).sum())
        Kd = K[:3 * nf, :3 * nf]
        scale = np.abs(Kd).max()
        assert np.abs(Kd - Kd.T).max() <= 1e-13 * scale
        w = np.linalg.eigvalsh(0.5 * (Kd + Kd.T))
        assert w.min() >= -1e-11 * scale
        assert int((w > 1e-9 * scale).sum()) == 6
        R = _rigid_modes(m.xyz[field[:nf]])
        assert np.abs(Kd @ R).max() <= 1e-10 * scale * max(1.0, np.abs(m.xyz).max())


def test_faces_sum_to_assembled_matrix():
    m = kuhn_beam(2, 1, 1, L=2.0, jitter=0.2, jitter_seed=1)
    o = Oracle(m.xyz, m.tets)
    fn, ft, fo = o.build_faces()
    nn = len(m.xyz)
    Kd = np.zeros((3 * nn, 3 * nn))
    for f in range(len(fn)):
        Kf, field = o.domain_stiffness(f, E, NU)
        nf = int((field >= 0).sum())
        idx = (3 * field[:nf, None] + np.arange(3)).ravel()
        Kd[np.ix_(idx, idx)] += Kf[:3 * nf, :3 * nf]
    _, rp, ci, va = o.assemble_fs(E, NU)
    Ka = np.zeros_like(Kd)
    for r in range(3 * nn):
        Ka[r, ci[rp[r]:rp[r + 1]]] += va[rp[r]:rp[r + 1]]
    assert np.abs(Kd - Ka).max() <= 1e-12 * np.abs(Ka).max()
