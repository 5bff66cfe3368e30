"""Pins of the CPU oracle against what PAPER.md and the mathematics fix (SURVEY.md 8(c) pin table).

Every oracle function is pinned here by something other than itself: values printed in the
paper (tests/golden), closed forms, invariants, special cases reducing to a textbook /
library routine, brute force on tiny inputs.  None of these tests touches the CUDA path.
"""
import itertools
import os
from fractions import Fraction

import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam, kuhn_counts
from oracle import Oracle, OracleError, csr_to_dense

E, NU = 1.0e6, 0.3
LAM = E * NU / ((1 + NU) * (1 - 2 * NU))
MU = E / (2 * (1 + NU))
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def two_tets():
    """Fig. 1: tets ABCD and ABCE share the interior face ABC (A,B,C,D,E = nodes 0..4)."""
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.2, 0.3, 1.0], [0.3, 0.2, -0.8]], float)
    tets = np.array([[0, 1, 2, 3], [0, 1, 2, 4]], np.int32)
    return xyz, tets


def unit_tet():
    return np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float), np.array([[0, 1, 2, 3]], np.int32)


def fem_gradients(X):
    """Textbook linear tet: columns of inv([1 x y z]) give N_I coefficients (independent of the oracle)."""
    M = np.hstack([np.ones((4, 1)), X])
    C = np.linalg.inv(M)
    return C[1:, :].T  # [4, 3] gradients of N_0..N_3


def textbook_cst_stiffness(X):
    """Constant-strain tet K_e = V B^T D B with numpy (Zienkiewicz-style layout)."""
    g = fem_gradients(X)
    V = abs(np.linalg.det(np.hstack([np.ones((4, 1)), X]))) / 6.0
    B = np.zeros((6, 12))
    for I in range(4):
        bx, by, bz = g[I]
        B[:, 3 * I:3 * I + 3] = [[bx, 0, 0], [0, by, 0], [0, 0, bz], [0, bz, by], [bz, 0, bx], [by, bx, 0]]
    D = np.zeros((6, 6))
    D[:3, :3] = LAM
    D[np.arange(3), np.arange(3)] = LAM + 2 * MU
    D[np.arange(3, 6), np.arange(3, 6)] = MU
    return V * B.T @ D @ B


def rigid_modes(xyz):
    n = xyz.shape[0]
    c = xyz.mean(axis=0)
    modes = []
    for a in range(3):
        r = np.zeros((n, 3))
        r[:, a] = 1.0
        modes.append(r.reshape(-1))
    for w in np.eye(3):
        modes.append(np.cross(w, xyz - c).reshape(-1))
    return modes


# ---------------------------------------------------------------- O1 volumes / validation
def test_eq10_volume_unit_tet():
    o = Oracle(*unit_tet())
    v = o.validate()
    assert abs(abs(v[0]) - 1.0 / 6.0) < 1e-16


def test_volume_sum_is_box_volume():
    for cfg in (1, 3):
        m = config_mesh(cfg)
        v = Oracle(m.xyz, m.tets).validate()
        assert abs(np.abs(v).sum() - 10.0) < 1e-11


def test_validation_errors():
    xyz, tets = unit_tet()
    with pytest.raises(OracleError) as e:
        Oracle(xyz, np.array([[0, 1, 2, 7]], np.int32)).validate()
    assert e.value.status == "invalid_arg"
    flat = xyz.copy()
    flat[3] = [0.3, 0.3, 0.0]
    with pytest.raises(OracleError) as e:
        Oracle(flat, tets).validate()
    assert e.value.status == "degenerate"
    with pytest.raises(OracleError) as e:
        Oracle(xyz, np.array([[0, 1, 1, 3]], np.int32)).validate()
    assert e.value.status == "degenerate"


# ---------------------------------------------------------------- O2 faces
def test_faces_single_and_two_tets():
    o = Oracle(*unit_tet())
    fn, ft, fo = o.build_faces()
    assert o.n_faces == 4 and o.n_interior == 0
    for f in range(4):
        assert ft[f, 1] == -1 and fo[f, 1] == -1
        assert set(fn[f]) | {fo[f, 0]} == {0, 1, 2, 3}  # remaining node = opposite vertex
    xyz, tets = two_tets()
    o = Oracle(xyz, tets)
    fn, ft, fo = o.build_faces()
    assert (o.n_faces, o.n_interior) == (7, 1)  # 1 interior + 6 exterior
    k = [f for f in range(7) if ft[f, 1] >= 0]
    assert len(k) == 1
    f = k[0]
    assert list(fn[f]) == [0, 1, 2] and list(ft[f]) == [0, 1] and list(fo[f]) == [3, 4]  # Fig. 1
    assert np.all(np.diff(fn[:, 0] * 100 + fn[:, 1] * 10 + fn[:, 2]) > 0)  # ascending (a,b,c)


def brute_force_faces(tets):
    """O(N_t^2) matching of tet faces by vertex sets (independent of the std::map oracle)."""
    faces = []
    for t, tet in enumerate(tets):
        for l in range(4):
            faces.append((frozenset(int(v) for i, v in enumerate(tet) if i != l), t, int(tet[l])))
    out = {}
    for i, (s, t, o) in enumerate(faces):
        owners = [(t2, o2) for (s2, t2, o2) in faces if s2 == s]
        out[tuple(sorted(s))] = sorted(owners)
    return out


def test_faces_brute_force_cfg1():
    m = config_mesh(1)
    o = Oracle(m.xyz, m.tets)
    fn, ft, fo = o.build_faces()
    bf = brute_force_faces(m.tets)
    assert len(bf) == o.n_faces
    assert [tuple(x) for x in fn] == sorted(bf.keys())
    for f in range(o.n_faces):
        owners = bf[tuple(fn[f])]
        if len(owners) == 1:
            assert (ft[f, 0], fo[f, 0], ft[f, 1], fo[f, 1]) == (owners[0][0], owners[0][1], -1, -1)
        else:
            assert len(owners) == 2
            assert (ft[f, 0], fo[f, 0], ft[f, 1], fo[f, 1]) == (*owners[0], *owners[1])


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_faces_closed_forms(cfg):
    m = config_mesh(cfg)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    c = kuhn_counts(*m.grid)
    assert (o.n_faces, o.n_interior) == (c["n_faces"], c["n_interior"])
    assert 4 * m.n_tets == 2 * o.n_interior + (o.n_faces - o.n_interior)


def test_faces_topology_error():
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1]], float)
    tets = np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]], np.int32)
    with pytest.raises(OracleError) as e:
        Oracle(xyz, tets).build_faces()
    assert e.value.status == "topology"


# ---------------------------------------------------------------- O3 smoothing domains (Table 1)
def read_table1():
    rows = {}
    with open(os.path.join(GOLDEN, "table1_shape_values.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            p = line.split()
            rows[p[0]] = tuple(Fraction(x) for x in p[1:])
    return rows


def test_table1_gauss_point_shape_values():
    xyz, tets = two_tets()
    o = Oracle(xyz, tets)
    fn, ft, fo = o.build_faces()
    f = int(np.nonzero(ft[:, 1] >= 0)[0][0])
    d = o.face_domain(f)
    table = read_table1()
    assert d["P"] == 6
    got = sorted(tuple(Fraction(round(v * 12), 12) for v in t[4:9]) for t in d["tri"])
    for t in d["tri"]:  # exact twelfths
        assert np.allclose(t[4:9] * 12, np.round(t[4:9] * 12), atol=1e-13)
    want = sorted(table[g] for g in ("g1", "g2", "g3", "g4", "g5", "g6"))
    assert got == want
    # partition of unity at every Gauss point
    assert np.allclose(d["tri"][:, 4:9].sum(axis=1), 1.0, atol=1e-15)
    # exterior face: P = 4 and the face's own triangle carries 1/3 on A, B, C
    fe = int(np.nonzero(ft[:, 1] < 0)[0][0])
    de = o.face_domain(fe)
    assert de["P"] == 4
    assert any(np.allclose(t[4:9], [1 / 3, 1 / 3, 1 / 3, 0, 0]) for t in de["tri"])


def test_domain_closed_surface_and_cone_volumes():
    m = kuhn_beam(3, 2, 2, jitter=0.2, jitter_seed=11)
    o = Oracle(m.xyz, m.tets)
    vol = np.abs(o.validate())
    fn, ft, fo = o.build_faces()
    total = 0.0
    for f in range(o.n_faces):
        d = o.face_domain(f)
        tri = d["tri"]
        assert np.allclose((tri[:, :1] * tri[:, 1:4]).sum(axis=0), 0.0, atol=1e-14)  # sum A_i n_i = 0
        # V_f = sum of quarter volumes of the owner tets (centroid at 1/4 height)
        expect = vol[ft[f, 0]] / 4 + (vol[ft[f, 1]] / 4 if ft[f, 1] >= 0 else 0.0)
        assert abs(d["Vf"] - expect) < 1e-14 * max(1.0, expect)
        total += d["Vf"]
    assert abs(total - 10.0) < 1e-12 and abs(vol.sum() - 10.0) < 1e-12  # sum V_f = |Omega| = L*W*H


# ---------------------------------------------------------------- O4 B-bar
def closed_form_bbar(xyz, tets, field, t0, t1):
    """Divergence theorem on each cone: b_I = sum_e (V_e/4) grad N_I^e / sum_e V_e/4."""
    num = np.zeros((5, 3))
    den = 0.0
    for t in (t0, t1):
        if t < 0:
            continue
        X = xyz[tets[t]]
        g = fem_gradients(X)
        V = abs(np.linalg.det(np.hstack([np.ones((4, 1)), X]))) / 6.0
        for I in range(5):
            if field[I] in tets[t]:
                num[I] += V / 4 * g[list(tets[t]).index(field[I])]
        den += V / 4
    return num / den


def test_eq7_equals_divergence_closed_form():
    m = kuhn_beam(4, 2, 2, jitter=0.25, jitter_seed=5)
    o = Oracle(m.xyz, m.tets)
    fn, ft, fo = o.build_faces()
    for f in range(o.n_faces):
        d = o.face_domain(f)
        bb = closed_form_bbar(m.xyz, m.tets, d["field"], ft[f, 0], ft[f, 1])
        scale = np.abs(bb).max()
        assert np.allclose(d["bbar"], bb, atol=1e-13 * scale), f
        assert np.allclose(d["bbar"].sum(axis=0), 0.0, atol=1e-13 * scale)  # sum_I b_I = 0


def test_linear_field_reproduction():
    """u = M x + t  =>  smoothed strain = sym(M) exactly."""
    m = kuhn_beam(3, 2, 2, jitter=0.2, jitter_seed=2)
    o = Oracle(m.xyz, m.tets)
    fn, ft, fo = o.build_faces()
    rng = np.random.default_rng(0)
    Mg = rng.normal(size=(3, 3))
    t = rng.normal(size=3)
    for f in range(0, o.n_faces, 7):
        d = o.face_domain(f)
        grad = np.zeros((3, 3))
        for I in range(5):
            if d["field"][I] < 0:
                continue
            u = Mg @ m.xyz[d["field"][I]] + t
            grad += np.outer(u, d["bbar"][I])  # du_a/dx_h = sum_I u_Ia b_Ih
        assert np.allclose(grad, Mg, atol=1e-12)


# ---------------------------------------------------------------- O4/O5 stiffness
def test_single_tet_fs_equals_fem_textbook():
    xyz = np.array([[0.1, 0.0, 0.2], [1.3, 0.1, 0.0], [0.2, 0.9, 0.1], [0.3, 0.2, 1.1]])
    tets = np.array([[0, 1, 2, 3]], np.int32)
    o = Oracle(xyz, tets)
    o.build_faces()
    lo, rp, ci, va = o.assemble_fs(E, NU)
    K = csr_to_dense(rp, ci, va, 12)
    Ke = textbook_cst_stiffness(xyz)
    assert np.allclose(K, Ke, atol=1e-12 * np.abs(Ke).max())
    lo, rp, ci, va = o.assemble_fem(E, NU)
    assert np.allclose(csr_to_dense(rp, ci, va, 12), Ke, atol=1e-12 * np.abs(Ke).max())
    assert o.last_coo_count() == 4 * 144  # 576 triplets


def test_eq12_triplet_count():
    counts = dict(l.split()[:2] for l in open(os.path.join(GOLDEN, "paper_counts.txt")) if l[0] != "#")
    xyz, tets = two_tets()
    o = Oracle(xyz, tets)
    o.build_faces()
    o.assemble_fs(E, NU)
    assert o.last_coo_count() == 1 * int(counts["eq12_interior_per_face"]) + 6 * int(
        counts["eq12_exterior_per_face"]) == 1089
    m = config_mesh(1)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    o.assemble_fs(E, NU)
    c = kuhn_counts(*m.grid)
    assert o.last_coo_count() == c["eq12_slots"]


@pytest.fixture(scope="module")
def cfg1_fs():
    m = config_mesh(1)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    lo, rp, ci, va = o.assemble_fs(E, NU)
    return m, o, rp, ci, va


def test_global_k_invariants(cfg1_fs):
    m, o, rp, ci, va = cfg1_fs
    n = 3 * m.n_nodes
    K = csr_to_dense(rp, ci, va, n)
    c = kuhn_counts(*m.grid)
    assert rp[-1] == c["nnz_fs"]  # nnz closed form (structural zeros kept)
    assert np.abs(K - K.T).max() <= 1e-12 * np.abs(K).max()
    for r in rigid_modes(m.xyz):
        assert np.abs(K @ r).max() <= 1e-10 * np.abs(K).sum(axis=1).max() * np.abs(r).max()
    ev = np.linalg.eigvalsh((K + K.T) / 2)
    assert ev[0] > -1e-9 * ev[-1]  # PSD
    assert np.sum(ev < 1e-9 * ev[-1]) == 6  # exactly the 6 rigid modes
    # block pattern = all field-node pairs
    for r in range(n):
        cols = ci[rp[r]:rp[r + 1]]
        assert np.all(np.diff(cols) > 0) and len(cols) % 3 == 0


def test_uniform_strain_energy_and_patch(cfg1_fs):
    """Linear u: u^T K u = |Omega| eps^T c eps, and K u = 0 at interior nodes (patch test)."""
    m, o, rp, ci, va = cfg1_fs
    m2 = kuhn_beam(4, 3, 3, jitter=0.2, jitter_seed=8)
    for mesh in (m, m2):
        oo = Oracle(mesh.xyz, mesh.tets)
        oo.build_faces()
        lo, rp2, ci2, va2 = oo.assemble_fs(E, NU)
        n = 3 * mesh.n_nodes
        K = csr_to_dense(rp2, ci2, va2, n)
        rng = np.random.default_rng(1)
        G = rng.normal(size=(3, 3))
        u = (mesh.xyz @ G.T).reshape(-1)
        eps = 0.5 * (G + G.T)
        ev = np.array([eps[0, 0], eps[1, 1], eps[2, 2], 2 * eps[1, 2], 2 * eps[0, 2], 2 * eps[0, 1]])
        D = np.zeros((6, 6))
        D[:3, :3] = LAM
        D[np.arange(3), np.arange(3)] = LAM + 2 * MU
        D[np.arange(3, 6), np.arange(3, 6)] = MU
        vol = mesh.dims[0] * mesh.dims[1] * mesh.dims[2]
        assert np.isclose(u @ K @ u, vol * ev @ D @ ev, rtol=1e-11)
        Ku = (K @ u).reshape(-1, 3)
        x = mesh.xyz
        L, W, H = mesh.dims
        interior = (x[:, 0] > 1e-12) & (x[:, 0] < L - 1e-12) & (x[:, 1] > 1e-12) & (x[:, 1] < W - 1e-12) & (
            x[:, 2] > 1e-12) & (x[:, 2] < H - 1e-12)
        assert interior.sum() > 0
        assert np.abs(Ku[interior]).max() <= 1e-10 * np.abs(K).max() * np.abs(u).max()


def test_loewner_fs_softer_than_fem():
    """K_FS <= K_FEM in the Loewner order (Jensen; SURVEY.md 8(c) O5 pin)."""
    m = kuhn_beam(4, 2, 2, jitter=0.2, jitter_seed=4)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    n = 3 * m.n_nodes
    Kfs = csr_to_dense(*o.assemble_fs(E, NU)[1:], n)
    Kfem = csr_to_dense(*o.assemble_fem(E, NU)[1:], n)
    ev = np.linalg.eigvalsh(Kfem - Kfs)
    assert ev[0] >= -1e-9 * np.abs(Kfem).max()
    # FEM-T4 companion pinned by the textbook element on every tet
    Kt = np.zeros((n, n))
    for t in m.tets:
        Ke = textbook_cst_stiffness(m.xyz[t])
        idx = np.concatenate([[3 * v, 3 * v + 1, 3 * v + 2] for v in t])
        Kt[np.ix_(idx, idx)] += Ke
    assert np.allclose(Kfem, Kt, atol=1e-12 * np.abs(Kt).max())
    # exterior faces each contribute 1/4 of their owner's FEM element: single tet already pinned;
    # the FS pattern is wider (field of interior faces adds the opposite pair)
    assert (np.abs(Kfs) > 0).sum() >= (np.abs(Kfem) > 0).sum()


def test_row_range_assembly_matches_full(cfg1_fs):
    m, o, rp, ci, va = cfg1_fs
    lo, rp2, ci2, va2 = o.assemble_fs(E, NU, 30, 47)
    assert lo == 90
    a, b = rp[90], rp[141]
    assert np.array_equal(rp2, rp[90:142] - a)
    assert np.array_equal(ci2, ci[a:b]) and np.array_equal(va2, va[a:b])
    o.assemble_fs(E, NU)  # restore full K for other users of the fixture


# ---------------------------------------------------------------- O6 BCs + O7 solve
def test_bc_modes_and_cholesky_agree():
    m = config_mesh(1)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    lo, rp0, ci0, va0 = o.assemble_fs(E, NU)
    u_elim = o.cholesky_eliminate(m.dirichlet, m.loads)
    rp, ci, va, f = o.apply_bc(m.dirichlet, m.loads, mode=0)
    u_mod = o.cholesky()
    fixed = np.zeros(3 * m.n_nodes, bool)
    for d in m.dirichlet:
        fixed[3 * d:3 * d + 3] = True
    assert np.all(u_mod[fixed] == 0.0)
    assert np.linalg.norm(u_mod - u_elim) <= 1e-11 * np.linalg.norm(u_elim)
    Kmod = csr_to_dense(rp, ci, va, 3 * m.n_nodes)
    # constrained rows/cols zero except the diagonal, diagonal kept
    K0 = csr_to_dense(rp0, ci0, va0, 3 * m.n_nodes)
    assert np.all(Kmod[fixed][:, ~fixed] == 0) and np.all(Kmod[~fixed][:, fixed] == 0)
    assert np.array_equal(np.diag(Kmod), np.diag(K0))
    u_pcg, rep = o.pcg(1e-10)
    assert rep["rel_residual"] <= 1e-10
    assert np.linalg.norm(u_pcg - u_mod) <= 1e-7 * np.linalg.norm(u_mod)
    assert np.isclose(u_pcg @ (Kmod @ u_pcg), f @ u_pcg, rtol=1e-8)  # energy identity
    o.assemble_fs(E, NU)
    o.apply_bc(m.dirichlet, m.loads, mode=1)
    u_pen = o.cholesky()
    en = lambda v: np.sqrt(max(v @ K0 @ v, 0.0))
    assert en(u_pen - u_elim) <= 1e-6 * en(u_elim)


def test_pcg_special_cases():
    xyz, tets = unit_tet()
    o = Oracle(xyz, tets)
    n = 12
    d = np.arange(1, n + 1, dtype=float)
    o.set_csr(np.arange(n + 1), np.arange(n, dtype=np.int32), d)
    o.apply_bc(np.zeros(0, np.int32), np.ones(n), mode=0)
    u, rep = o.pcg(1e-12)
    assert rep["iterations"] == 1 and np.allclose(u, 1.0 / d, rtol=1e-15)  # Jacobi exact on diagonal K
    rng = np.random.default_rng(3)
    A = rng.normal(size=(n, n))
    A = A @ A.T + n * np.eye(n)
    b = rng.normal(size=n)
    rows, cols = np.nonzero(np.ones((n, n)))
    o.set_csr(np.arange(0, n * n + 1, n), cols.astype(np.int32), A.reshape(-1))
    o.apply_bc(np.zeros(0, np.int32), b, mode=0)
    u, rep = o.pcg(1e-13)
    x = np.linalg.solve(A, b)
    assert np.linalg.norm(u - x) <= 1e-11 * np.linalg.norm(x) and rep["iterations"] <= n + 2
    assert np.allclose(o.cholesky(), x, rtol=1e-12)
    o.apply_bc(np.zeros(0, np.int32), np.zeros(n), mode=0)
    u, rep = o.pcg()
    assert rep["iterations"] == 0 and np.all(u == 0)


@pytest.mark.parametrize("cfg", [1, 2])
def test_fs_tip_deflection_exceeds_fem(cfg):
    """K_FS <= K_FEM => f^T K_FS^-1 f >= f^T K_FEM^-1 f; with the uniform tip load that is the
    mean tip u_z (reading Q15).  Also the FS value stays below Euler-Bernoulli + Timoshenko."""
    m = config_mesh(cfg)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    tip = []
    for asm in (o.assemble_fs, o.assemble_fem):
        asm(E, NU)
        o.apply_bc(m.dirichlet, m.loads, 0)
        u, rep = o.pcg(1e-10)
        tip.append(-u.reshape(-1, 3)[m.tip, 2].mean())
    fs, fem = tip
    assert fs >= fem > 0
    eb = 1.0 * 10.0 ** 3 / (3 * E * (1.0 / 12.0))
    assert fs < 1.03 * (eb + 3.06e-5)


def test_table5_dense_sizes_pin_dof_layout():
    """Table 5: dense size = (3 N_n)^2 * 8 B — 3 dofs per node, fp64 (reading Q12)."""
    for line in open(os.path.join(GOLDEN, "paper_counts.txt")):
        if line.startswith("table5_dense"):
            _, nn, gb = line.split()
            assert abs((3 * int(nn)) ** 2 * 8 / 2 ** 30 - float(gb)) < 0.006
