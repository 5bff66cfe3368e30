"""GPU (sm_100a, through the C ABI) vs the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): faces / adjacency / row_ptr / col_idx bit-exact;
CSR values within 1e-12 * max|K|; displacements within 1e-7 relative L2 at PCG residual 1e-10.
Full-size configs (4, 5) are checked on sampled rows the oracle computes one by one and on
properties that hold at any size.
"""
import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam, kuhn_counts
from oracle import Oracle

pytestmark = pytest.mark.gpu

E, NU = 1.0e6, 0.3
VAL_TOL = 1e-12
U_TOL = 1e-7


@pytest.fixture(scope="module")
def fs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2001_08849_b200 import FsFem, load_library
    load_library()
    return FsFem


def gpu_faces(FsFem, m):
    g = FsFem()
    g.build_faces(m.xyz, m.tets)
    return g, g.get_faces()


def check_faces(FsFem, m):
    o = Oracle(m.xyz, m.tets)
    ofn, oft, ofo = o.build_faces()
    g, (fn, ft, fo) = gpu_faces(FsFem, m)
    assert (g.n_faces, g.n_interior) == (o.n_faces, o.n_interior)
    assert np.array_equal(fn, ofn) and np.array_equal(ft, oft) and np.array_equal(fo, ofo)
    return g, o


def small_meshes():
    yield "cfg1", config_mesh(1)
    yield "cfg2", config_mesh(2)
    yield "ragged", kuhn_beam(7, 3, 5, L=3.0, jitter=0.2, jitter_seed=17)
    yield "ragged_perm", kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8, tet_perm_seed=9)
    yield "cfg3", config_mesh(3)


@pytest.mark.parametrize("name,m", list(small_meshes()), ids=[n for n, _ in small_meshes()])
def test_faces_bit_exact(fs, name, m):
    check_faces(fs, m)


def test_faces_hand_meshes_and_errors(fs):
    from paper_2001_08849_b200 import FsfemError
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.2, 0.3, 1.0], [0.3, 0.2, -0.8]], float)
    g = fs()
    assert g.build_faces(xyz, np.array([[0, 1, 2, 3]], np.int32)) == (4, 0)
    assert g.build_faces(xyz, np.array([[0, 1, 2, 3], [0, 1, 2, 4]], np.int32)) == (7, 1)
    fn, ft, fo = g.get_faces()
    k = int(np.nonzero(ft[:, 1] >= 0)[0][0])
    assert list(fn[k]) == [0, 1, 2] and list(ft[k]) == [0, 1] and list(fo[k]) == [3, 4]
    bad = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1]], float)
    with pytest.raises(FsfemError) as e:
        g.build_faces(bad, np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]], np.int32))
    assert e.value.status == "TOPOLOGY"
    with pytest.raises(FsfemError) as e:
        g.build_faces(xyz, np.array([[0, 1, 2, 9]], np.int32))
    assert e.value.status == "INVALID_ARG"
    flat = xyz.copy()
    flat[3] = [0.3, 0.3, 0.0]
    with pytest.raises(FsfemError) as e:
        g.build_faces(flat, np.array([[0, 1, 2, 3]], np.int32))
    assert e.value.status == "DEGENERATE"
    with pytest.raises(FsfemError) as e:
        g.assemble_csr(E, NU)  # failed build leaves the context without faces
    assert e.value.status == "STATE"


def check_csr(g, o, node_lo=0, node_hi=None):
    """Compare GPU CSR rows of nodes [node_lo, node_hi) with the oracle's."""
    c = g.get_csr()
    node_hi = g.n_nodes if node_hi is None else node_hi
    lo, orp, oci, ova = o.assemble_fs(E, NU, node_lo, node_hi)
    r0, r1 = 3 * node_lo, 3 * node_hi
    rp = c.row_ptr[r0:r1 + 1] - c.row_ptr[r0]
    assert np.array_equal(rp, orp)
    a, b = c.row_ptr[r0], c.row_ptr[r1]
    assert np.array_equal(c.col_idx[a:b], oci)
    kmax = np.abs(ova).max()
    err = np.abs(c.vals[a:b] - ova).max()
    assert err <= VAL_TOL * kmax, (err, kmax)
    return c, kmax


@pytest.mark.parametrize("name,m", [x for x in small_meshes() if x[0] != "cfg3"],
                         ids=[n for n, _ in small_meshes() if n != "cfg3"])
def test_csr_parity_small(fs, name, m):
    g, o = check_faces(fs, m)
    g.assemble_csr(E, NU)
    assert g.nnz == o.assemble_fs(E, NU)[1][-1]
    check_csr(g, o)
    if name.startswith("cfg"):
        assert g.nnz == kuhn_counts(*m.grid)["nnz_fs"]


def test_csr_parity_cfg3_rows(fs):
    m = config_mesh(3)
    g, o = check_faces(fs, m)
    g.assemble_csr(E, NU)
    check_csr(g, o, 0, 3000)          # first tile run (clamped end)
    check_csr(g, o, 20000, 20777)     # interior, ragged count
    check_csr(g, o, m.n_nodes - 1500, m.n_nodes)  # tip end


def solve_both(fs, m, mode=0):
    g, o = check_faces(fs, m)
    g.assemble_csr(E, NU)
    o.assemble_fs(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1), mode)
    orp, oci, ova, of = o.apply_bc(m.dirichlet, m.loads, mode)
    c = g.get_csr()
    assert np.array_equal(c.row_ptr, orp) and np.array_equal(c.col_idx, oci)
    assert np.abs(c.vals - ova).max() <= VAL_TOL * np.abs(ova).max()
    u, rep = g.pcg_solve(rel_tol=1e-10)
    uo, orep = o.pcg(1e-10)
    return g, o, u, rep, uo, orep


@pytest.mark.parametrize("name,m", [x for x in small_meshes() if x[0] != "cfg3"],
                         ids=[n for n, _ in small_meshes() if n != "cfg3"])
def test_solve_parity(fs, name, m):
    g, o, u, rep, uo, orep = solve_both(fs, m)
    assert rep["converged"] == 1 and rep["rel_residual"] <= 1e-10
    assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
    fixed = np.zeros(3 * m.n_nodes, bool)
    for d in m.dirichlet:
        fixed[3 * d:3 * d + 3] = True
    assert np.all(u[fixed] == 0.0)
    if name == "cfg1":
        uc = o.cholesky()
        assert np.linalg.norm(u - uc) <= U_TOL * np.linalg.norm(uc)
    # Iteration counts are not a parity quantity (rounding order differs: GPU FMA, symmetric-storage
    # SpMV, tree dots); they must still be close.  cfg1 (297 dofs) needs ~n iterations, where CG
    # is most sensitive to rounding.
    assert abs(rep["iterations"] - orep["iterations"]) <= max(3, 0.05 * orep["iterations"])


def test_penalty_mode(fs):
    m = config_mesh(1)
    g, o, u, rep, uo, orep = solve_both(fs, m, mode=1)
    assert np.linalg.norm(u - uo) <= 1e-6 * np.linalg.norm(uo)


def test_determinism_and_warm_start(fs):
    m = kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8, tet_perm_seed=9)
    outs = []
    for _ in range(2):
        g = fs()
        g.build_faces(m.xyz, m.tets)
        g.assemble_csr(E, NU)
        v1 = g.get_csr().vals.copy()
        g.assemble_csr(E, NU)  # numeric-only re-assembly
        v2 = g.get_csr().vals.copy()
        assert np.array_equal(v1, v2)
        g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        u, rep = g.pcg_solve()
        outs.append((v1, u))
        u2, rep2 = g.pcg_solve(u0=u)  # warm start from the solution: converges immediately
        assert rep2["iterations"] <= 2
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_state_machine(fs):
    from paper_2001_08849_b200 import FsfemError
    g = fs()
    for call in (lambda: g.assemble_csr(E, NU), lambda: g.pcg_solve()):
        with pytest.raises(FsfemError) as e:
            call()
        assert e.value.status == "STATE"
    m = config_mesh(1)
    g.build_faces(m.xyz, m.tets)
    with pytest.raises(FsfemError) as e:
        g.assemble_csr(E, 0.5)
    assert e.value.status == "INVALID_ARG"


def test_device_pointers_accepted(fs):
    import torch
    from paper_2001_08849_b200 import fsfem_build_faces, fsfem_get_faces
    m = config_mesh(2)
    g = fs()
    xyz = torch.from_numpy(m.xyz).cuda()
    tets = torch.from_numpy(m.tets).cuda()
    nf, ni = fsfem_build_faces(g.ctx, xyz, tets)
    fn = torch.empty((nf, 3), dtype=torch.int32, device="cuda")
    fsfem_get_faces(g.ctx, fn, None, None)
    o = Oracle(m.xyz, m.tets)
    ofn, _, _ = o.build_faces()
    assert np.array_equal(fn.cpu().numpy(), ofn)


# ---------------------------------------------------------------- full-size configs (bench launch config)
@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_faces_and_sampled_rows(fs, cfg):
    m = config_mesh(cfg)
    g = fs()
    nf, ni = g.build_faces(m.xyz, m.tets)
    c = kuhn_counts(*m.grid)
    assert (nf, ni) == (c["n_faces"], c["n_interior"])
    fn, ft, fo = g.get_faces()
    # properties at any size: strictly ascending keys, owners contain the face, opp is the 4th node
    key = (fn[:, 0].astype(np.int64) << 42) | (fn[:, 1].astype(np.int64) << 21) | fn[:, 2]
    assert np.all(np.diff(key) > 0) and np.all(fn[:, 0] < fn[:, 1]) and np.all(fn[:, 1] < fn[:, 2])
    for k in (0, 1):
        sel = ft[:, k] >= 0
        tt = m.tets[ft[sel, k]]
        for a in range(3):
            assert np.all(np.any(tt == fn[sel, a:a + 1], axis=1))
        assert np.all(np.any(tt == fo[sel, k:k + 1], axis=1))
        assert not np.any(np.any(fn[sel] == fo[sel, k:k + 1], axis=1))
    assert np.all(ft[ft[:, 1] >= 0, 0] < ft[ft[:, 1] >= 0, 1])
    g.assemble_csr(E, NU)
    assert g.nnz == c["nnz_fs"]
    o = Oracle(m.xyz, m.tets)
    ofn, oft, ofo = o.build_faces()
    # bit-exact against the oracle's map-based face table at full size
    assert np.array_equal(fn, ofn) and np.array_equal(ft, oft) and np.array_equal(fo, ofo)
    del ofn, oft, ofo
    rng = np.random.default_rng(cfg)
    for lo in [0, m.n_nodes - 400, *rng.integers(0, m.n_nodes - 300, 2)]:
        check_csr(g, o, int(lo), int(lo) + 257)


def test_cfg4_solution_properties(fs):
    """cfg4 at full size: residual, energy identity, Euler-Bernoulli within 3% (north star)."""
    m = config_mesh(4)
    g = fs()
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve(rel_tol=1e-10)
    assert rep["converged"] == 1
    assert rep["true_rel_residual"] < 1e-7
    f = m.loads.reshape(-1).copy()
    Ku = g.spmv(u)
    assert np.isclose(u @ Ku, f @ u, rtol=1e-8)
    tip = -u.reshape(-1, 3)[m.tip, 2].mean()
    eb = 1.0 * 10.0 ** 3 / (3 * E * (1.0 / 12.0))
    assert abs(tip - eb) <= 0.03 * eb, (tip, eb)


# ---------------------------------------------------------------- row partition (multi-GPU layout)
@pytest.mark.parametrize("nranks", [2, 3])
def test_row_partition_contexts(fs, nranks):
    """Partition-only contexts (include/fsfem.h) hold rank r's rows on one GPU: halo blocks
    (columns below the rank's range) are stored, the rest of the lower half is read transposed.
    Each rank's CSR rows, SpMV rows and BC-modified rows must equal the oracle's."""
    from paper_2001_08849_b200 import FsfemError
    m = kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8, tet_perm_seed=9)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    _, _, _, full_vals = o.assemble_fs(E, NU)
    kmax = np.abs(full_vals).max()
    x = np.random.default_rng(nranks).standard_normal(3 * m.n_nodes)
    q_ref = o.spmv(x)
    orp_bc, oci_bc, ova_bc, _ = o.apply_bc(m.dirichlet, m.loads, 0)
    for r in range(nranks):
        g = fs()
        g.comm_init(None, r, nranks)
        g.build_faces(m.xyz, m.tets)
        rng = g.partition()
        assert rng[0] == 0 and rng[-1] == m.n_nodes and np.all(np.diff(rng) > 0)
        lo, hi = int(rng[r]), int(rng[r + 1])
        rb, nr, nnz = g.assemble_csr(E, NU)
        assert (rb, nr) == (3 * lo, 3 * (hi - lo))
        c = g.get_csr()
        _, orp, oci, ova = o.assemble_fs(E, NU, lo, hi)
        assert np.array_equal(c.row_ptr, orp) and np.array_equal(c.col_idx, oci)
        assert np.abs(c.vals - ova).max() <= VAL_TOL * kmax
        q = g.spmv(x)
        scale = kmax * np.abs(x).max()
        assert np.abs(q[3 * lo:3 * hi] - q_ref[3 * lo:3 * hi]).max() <= 1e-11 * scale
        g.apply_bc(m.dirichlet, m.loads.reshape(-1), 0)
        c = g.get_csr()
        a, b = orp_bc[3 * lo], orp_bc[3 * hi]
        assert np.array_equal(c.col_idx, oci_bc[a:b])
        assert np.abs(c.vals - ova_bc[a:b]).max() <= VAL_TOL * kmax
        with pytest.raises(FsfemError) as e:
            g.pcg_solve()
        assert e.value.status == "STATE"


# ---------------------------------------------------------------- full-size displacements vs the oracle
def _gpu_solve(fs, m):
    g = fs()
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve(rel_tol=1e-10)
    return g, u, rep


def _golden(cfg):
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"oracle_cfg{cfg}.json")))


def test_cfg3_displacements_match_oracle(fs):
    """cfg3 (jittered, 134k dofs): the whole u against the oracle's full solve
    (tests/golden/oracle_cfg3_u.npy, written by scripts/oracle_full_solve.py from oracle/ only)."""
    import os
    m = config_mesh(3)
    g, u, rep = _gpu_solve(fs, m)
    uo = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg3_u.npy"))
    gold = _golden(3)
    assert rep["converged"] == 1 and rep["rel_residual"] <= 1e-10
    assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
    f = m.loads.reshape(-1)
    assert abs(f @ u - gold["f_dot_u"]) <= 1e-8 * abs(gold["f_dot_u"])
    assert abs(rep["iterations"] - gold["pcg"]["iterations"]) <= 0.05 * gold["pcg"]["iterations"]


def test_cfg4_displacements_match_oracle(fs):
    """cfg4 (bench workload): the WHOLE u against the oracle's full solve
    (tests/golden/oracle_cfg4_u.npy, written by scripts/oracle_full_solve.py 4 from oracle/ only:
    ||u - u_ora||_2 <= 1e-7 ||u_ora||_2), plus compliance, tip deflection and the json samples."""
    import os
    m = config_mesh(4)
    g, u, rep = _gpu_solve(fs, m)
    gold = _golden(4)
    assert rep["converged"] == 1
    uo = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg4_u.npy"))
    assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
    f = m.loads.reshape(-1)
    assert abs(f @ u - gold["f_dot_u"]) <= 1e-8 * abs(gold["f_dot_u"])
    tip = u.reshape(-1, 3)[m.tip, 2].mean()
    assert abs(tip - gold["tip_mean_uz"]) <= 1e-7 * abs(gold["tip_mean_uz"])
    idx = np.asarray(gold["u_sample_idx"])
    assert np.abs(u[idx] - np.asarray(gold["u_sample"])).max() <= U_TOL * gold["u_norm"]
    assert abs(np.linalg.norm(u) - gold["u_norm"]) <= U_TOL * gold["u_norm"]


def test_cfg5_solution_properties(fs):
    """cfg5 (9.8M tets, jittered, randomly relabelled; no full oracle solve exists -- SURVEY R4):
    convergence, true residual, energy identity and the beam deflection between the
    Euler-Bernoulli value and the Timoshenko one (+3%)."""
    m = config_mesh(5)
    g, u, rep = _gpu_solve(fs, m)
    assert rep["converged"] == 1 and rep["rel_residual"] <= 1e-10
    assert rep["true_rel_residual"] < 1e-6
    f = m.loads.reshape(-1)
    Ku = g.spmv(u)
    assert np.isclose(u @ Ku, f @ u, rtol=1e-8)
    tip = -u.reshape(-1, 3)[m.tip, 2].mean()
    eb = 1.0 * 10.0 ** 3 / (3 * E * (1.0 / 12.0))
    assert 0.97 * eb <= tip <= 1.03 * 4.031e-3, (tip, eb)
    fixed = np.repeat(np.isin(np.arange(m.n_nodes), m.dirichlet), 3)
    assert np.all(u[fixed] == 0.0)


def test_cfg5_displacements_match_oracle(fs):
    """cfg5 (9.8M tets, randomly relabelled: the library renumbers internally and translates
    back): the WHOLE u against the oracle's full solve (tests/golden/oracle_cfg5_u.npy, written by
    scripts/oracle_full_solve.py 5 8 --u-only: oracle/ only, ~1.5 h on 8 CPU threads), plus
    compliance, tip deflection and the 4096 sampled dofs of tests/golden/oracle_cfg5.json."""
    import os
    m = config_mesh(5)
    g, u, rep = _gpu_solve(fs, m)
    gold = _golden(5)
    assert rep["converged"] == 1 and rep["reordered"] == 1
    uo = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg5_u.npy"))
    assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
    f = m.loads.reshape(-1)
    assert abs(f @ u - gold["f_dot_u"]) <= 1e-8 * abs(gold["f_dot_u"])
    tip = u.reshape(-1, 3)[m.tip, 2].mean()
    assert abs(tip - gold["tip_mean_uz"]) <= 1e-7 * abs(gold["tip_mean_uz"])
    idx = np.asarray(gold["u_sample_idx"])
    assert np.abs(u[idx] - np.asarray(gold["u_sample"])).max() <= U_TOL * gold["u_norm"]
    assert abs(np.linalg.norm(u) - gold["u_norm"]) <= U_TOL * gold["u_norm"]
    assert abs(rep["iterations"] - gold["pcg"]["iterations"]) <= 0.05 * gold["pcg"]["iterations"]


# ---------------------------------------------------------------- error paths and edge cases
def test_not_converged_reports_and_writes_u(fs):
    from paper_2001_08849_b200 import fsfem_pcg_solve
    m = config_mesh(2)
    g = fs()
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u = np.zeros(3 * m.n_nodes)
    rep = fsfem_pcg_solve(g.ctx, u, True, 1e-10, 7, allow_not_converged=True)
    assert rep["status"] == "NOT_CONVERGED" and rep["iterations"] == 7 and rep["converged"] == 0
    assert np.linalg.norm(u) > 0 and rep["rel_residual"] > 1e-10
    # the same 7 iterations as the start of a full solve: deterministic prefix
    g2 = fs()
    g2.build_faces(m.xyz, m.tets)
    g2.assemble_csr(E, NU)
    g2.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u2 = np.zeros(3 * m.n_nodes)
    fsfem_pcg_solve(g2.ctx, u2, True, 1e-10, 7, allow_not_converged=True)
    assert np.array_equal(u, u2)


def test_invalid_arguments(fs):
    from paper_2001_08849_b200 import FsfemError
    m = config_mesh(1)
    g = fs()
    with pytest.raises(FsfemError) as e:
        g.build_faces(m.xyz, m.tets[:0])
    assert e.value.status == "INVALID_ARG"
    g.build_faces(m.xyz, m.tets)
    for bad in ((0.0, 0.3), (-1.0, 0.3), (E, 0.5), (E, -1.0)):
        with pytest.raises(FsfemError) as e:
            g.assemble_csr(*bad)
        assert e.value.status == "INVALID_ARG"
    g.assemble_csr(E, NU)
    with pytest.raises(FsfemError) as e:
        g.apply_bc(np.array([0, m.n_nodes], np.int32), m.loads.reshape(-1))
    assert e.value.status == "INVALID_ARG"
    with pytest.raises(FsfemError) as e:
        g.apply_bc(m.dirichlet, m.loads.reshape(-1), 7)
    assert e.value.status == "INVALID_ARG"


def test_outputs_to_device_buffers(fs):
    """get_csr / pcg_solve with CUDA tensors as outputs (no host round trip) equal the host path."""
    import torch
    from paper_2001_08849_b200 import fsfem_get_csr, fsfem_pcg_solve
    m = config_mesh(2)
    g = fs()
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    c = g.get_csr()
    rp = torch.empty(g.n_rows + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(g.nnz, dtype=torch.int32, device="cuda")
    va = torch.empty(g.nnz, dtype=torch.float64, device="cuda")
    fsfem_get_csr(g.ctx, rp, ci, va)
    assert np.array_equal(rp.cpu().numpy(), c.row_ptr) and np.array_equal(ci.cpu().numpy(), c.col_idx)
    assert np.array_equal(va.cpu().numpy(), c.vals)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u_h, _ = g.pcg_solve()
    u_d = torch.zeros(3 * m.n_nodes, dtype=torch.float64, device="cuda")
    fsfem_pcg_solve(g.ctx, u_d, True, 1e-10, 0)
    assert np.array_equal(u_d.cpu().numpy(), u_h)


def test_unreferenced_node_is_rejected_by_bcs(fs):
    """A node in no tet has an empty row: the Jacobi preconditioner cannot be formed (BREAKDOWN
    from apply_bc), unless the node is clamped."""
    from paper_2001_08849_b200 import FsfemError
    m = config_mesh(1)
    xyz = np.vstack([m.xyz, [[20.0, 0.0, 0.0]]])
    g = fs()
    g.build_faces(xyz, m.tets)
    g.assemble_csr(E, NU)
    loads = np.zeros(3 * (m.n_nodes + 1))
    loads[:3 * m.n_nodes] = m.loads.reshape(-1)
    with pytest.raises(FsfemError) as e:
        g.apply_bc(m.dirichlet, loads)
    assert e.value.status == "BREAKDOWN"


def test_full_pipeline_bitwise_reproducible_cfg3(fs):
    """Two complete runs (faces, pattern, assembly, BCs, PCG) on cfg3 give byte-identical CSR values
    and displacements: every reduction has a fixed order (Q26), no atomics on values."""
    m = config_mesh(3)
    outs = []
    for _ in range(2):
        g = fs()
        g.build_faces(m.xyz, m.tets)
        g.assemble_csr(E, NU)
        v = g.get_csr(with_pattern=False).vals.copy()
        g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        u, rep = g.pcg_solve()
        outs.append((v, u, rep["iterations"]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1]) and outs[0][2] == outs[1][2]
