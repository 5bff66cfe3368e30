"""Cluster PCG (fsfem_set_loop FSFEM_LOOP_CLUSTER; the default FSFEM_LOOP_AUTO picks it for small
meshes): the whole Jacobi-PCG recurrence (S8-S9) in one launch of one thread-block cluster, with
cluster-wide reductions over distributed shared memory.  Same bars as every solve: converged at
rel_tol 1e-10, u within 1e-7 relative L2 of the oracle's solve; plus bitwise reproducibility, the
AUTO selection rule and the fallback to the host loop where the kernel does not apply."""
import os

import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam
from oracle import Oracle

pytestmark = pytest.mark.gpu

E, NU = 1.0e6, 0.3
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
LOOP_DEVICE, LOOP_HOST, LOOP_CLUSTER, LOOP_AUTO = 0, 1, 2, 3


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2001_08849_b200 as P
    P.load_library()
    return P


def _oracle_u(m):
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    o.assemble_fs(E, NU)
    o.apply_bc(m.dirichlet, m.loads, 0)
    u, _ = o.pcg(1e-10)
    return u


def _solve(P, m, loop, **kw):
    g = P.FsFem()
    try:
        g.set_loop(loop)
        g.build_faces(m.xyz, m.tets)
        g.assemble_csr(E, NU)
        g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        return g.pcg_solve(**kw)
    finally:
        g.close()


MESHES = {"cfg1": lambda: config_mesh(1), "cfg2": lambda: config_mesh(2),
          "ragged_perm": lambda: kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8,
                                           tet_perm_seed=9)}


@pytest.mark.parametrize("name", list(MESHES))
def test_cluster_matches_oracle(P, name):
    m = MESHES[name]()
    u, rep = _solve(P, m, LOOP_AUTO if name != "cfg2" else LOOP_CLUSTER, rel_tol=1e-10)
    assert rep["pcg_loop"] == LOOP_CLUSTER  # AUTO picks it for cfg1 and the ragged mesh (< 8000 blocks)
    assert rep["converged"] == 1 and rep["rel_residual"] <= 1e-10
    assert rep["true_rel_residual"] <= max(1e-10, rep["residual_floor"])
    uo = _oracle_u(m)
    assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)
    fixed = np.repeat(np.isin(np.arange(m.n_nodes), m.dirichlet), 3)
    assert np.all(u[fixed] == 0.0)
    # bitwise reproducible, and the same recurrence as the multi-kernel loop up to rounding
    u2, rep2 = _solve(P, m, LOOP_CLUSTER, rel_tol=1e-10)
    assert np.array_equal(u, u2) and rep2["iterations"] == rep["iterations"]
    uh, reph = _solve(P, m, LOOP_HOST, rel_tol=1e-10)
    assert reph["pcg_loop"] == LOOP_HOST
    assert abs(rep["iterations"] - reph["iterations"]) <= max(2, 0.02 * reph["iterations"])


def test_cluster_on_cfg3_matches_oracle_golden(P):
    m = config_mesh(3)
    u, rep = _solve(P, m, LOOP_CLUSTER, rel_tol=1e-10)
    assert rep["pcg_loop"] == LOOP_CLUSTER and rep["converged"] == 1
    uo = np.load(os.path.join(GOLDEN, "oracle_cfg3_u.npy"))
    assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)
    _, rep_auto = _solve(P, m, LOOP_AUTO, rel_tol=1e-10, max_iter=3, allow_not_converged=True)
    assert rep_auto["pcg_loop"] == LOOP_HOST  # 1.1M blocks: above the AUTO threshold
    _, rep_auto = _solve(P, config_mesh(2), LOOP_AUTO, rel_tol=1e-10, max_iter=3, allow_not_converged=True)
    assert rep_auto["pcg_loop"] == LOOP_HOST  # cfg2, 74k blocks: the multi-kernel loop is faster


def test_cluster_iteration_budget_and_warm_start(P):
    m = config_mesh(2)
    u, rep = _solve(P, m, LOOP_CLUSTER, rel_tol=1e-10, max_iter=7, allow_not_converged=True)
    assert rep["converged"] == 0 and rep["iterations"] == 7 and rep["pcg_loop"] == LOOP_CLUSTER
    g = P.FsFem()
    g.set_loop(LOOP_CLUSTER)
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u1, r1 = g.pcg_solve(rel_tol=1e-10)
    u2, r2 = g.pcg_solve(u0=u1, rel_tol=1e-10)  # warm start from the solution
    assert r2["converged"] == 1 and r2["iterations"] <= 5  # the true residual of u1 is near the tolerance
    assert np.linalg.norm(u2 - u1) <= 1e-9 * np.linalg.norm(u1)
    g.close()


def test_cluster_request_falls_back_where_not_applicable(P):
    import torch
    m = config_mesh(2)
    stream = torch.cuda.Stream()
    gs = [P.FsFem(stream=stream.cuda_stream) for _ in range(2)]
    try:
        P.fsfem_comm_init_loopback([g.ctx for g in gs])
        for g in gs:
            g.nranks = 2
            g.set_loop(LOOP_CLUSTER)
            g.build_faces(m.xyz, m.tets)
            g.assemble_csr(E, NU)
            g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        u, rep = gs[0].pcg_solve(rel_tol=1e-10)
        assert rep["pcg_loop"] == LOOP_HOST and rep["converged"] == 1
    finally:
        for g in gs:
            g.close()
    g = P.FsFem()
    g.set_loop(LOOP_CLUSTER)
    g.set_pcg_variant(1)  # single-reduction recurrence: multi-kernel path
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve(rel_tol=1e-10)
    assert rep["pcg_loop"] == LOOP_HOST and rep["converged"] == 1
    g.close()
