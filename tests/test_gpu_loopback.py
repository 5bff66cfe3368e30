"""Multi-rank PCG executed on one GPU: the loopback group (fsfem_comm_init_loopback, SURVEY.md §4
"simulated partition").  G contexts in one process are ranks 0..G-1 of a
row partition (nnz-balanced node ranges); fsfem_pcg_solve runs every rank's
kernels and the multi-rank collectives (all-gather of dot partials + combine, all-gather(v) or
halo exchange of the search direction, deterministic chunk partials) as device copies.

Bars: u within 1e-7 relative L2 of the oracle's solve for every recurrence and exchange variant;
with deterministic dots (fsfem_set_deterministic) u is bit-identical for G = 1, 2, 3, 4.
"""
import os

import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam

pytestmark = pytest.mark.gpu

E, NU = 1.0e6, 0.3
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2001_08849_b200 as P
    P.load_library()
    return P


def solve_group(P, m, G, variant=0, exchange=0, det=False, rel_tol=1e-10, overlap=False):
    import torch
    stream = torch.cuda.Stream()
    gs = [P.FsFem(device=0, stream=stream.cuda_stream) for _ in range(G)]
    try:
        if G > 1:
            P.fsfem_comm_init_loopback([g.ctx for g in gs])
            for g in gs:
                g.nranks = G
        for g in gs:
            if det:
                g.set_deterministic(True)
            g.set_exchange(exchange)
            g.set_pcg_variant(variant)
            g.set_overlap(overlap)
            g.build_faces(m.xyz, m.tets)
            g.assemble_csr(E, NU)
            g.apply_bc(m.dirichlet, m.loads.reshape(-1))
        rng = gs[0].partition()
        u, rep = gs[G - 1].pcg_solve(rel_tol=rel_tol)  # any rank drives the group
        torch.cuda.synchronize()
        return u, rep, rng
    finally:
        for g in gs:
            g.close()


def test_partition_ranges_balanced(lib):
    m = config_mesh(3)
    for G, det in ((2, False), (3, False), (4, True)):
        import torch
        stream = torch.cuda.Stream()
        gs = [lib.FsFem(device=0, stream=stream.cuda_stream) for _ in range(G)]
        lib.fsfem_comm_init_loopback([g.ctx for g in gs])
        for g in gs:
            g.nranks = G
            if det:
                g.set_deterministic(True)
            g.build_faces(m.xyz, m.tets)
        rngs = [g.partition() for g in gs]
        for r in rngs[1:]:
            assert np.array_equal(r, rngs[0])
        rng = rngs[0]
        assert rng[0] == 0 and rng[-1] == m.n_nodes and np.all(np.diff(rng) > 0)
        align = 256 if det else 32
        assert np.all(rng[1:-1] % align == 0)
        # balanced by node-face incidences (each node: number of faces whose field holds it)
        fn, _, fo = gs[0].get_faces()
        w = np.bincount(np.concatenate([fn.ravel(), fo[fo >= 0]]), minlength=m.n_nodes)
        share = np.array([w[a:b].sum() for a, b in zip(rng[:-1], rng[1:])]) / w.sum()
        assert np.abs(share - 1.0 / G).max() <= 0.02
        for g in gs:
            g.close()


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("variant,exchange", [(0, 0), (0, 1), (1, 0), (1, 1)],
                         ids=["std-allgather", "std-halo", "single-allgather", "single-halo"])
def test_loopback_solve_matches_oracle_cfg3(lib, G, variant, exchange):
    m = config_mesh(3)
    uo = np.load(os.path.join(GOLDEN, "oracle_cfg3_u.npy"))
    u, rep, rng = solve_group(lib, m, G, variant, exchange)
    assert rep["converged"] == 1 and rep["rel_residual"] <= 1e-10
    assert rep["true_rel_residual"] <= max(1e-10, rep["residual_floor"])
    assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)
    fixed = np.repeat(np.isin(np.arange(m.n_nodes), m.dirichlet), 3)
    assert np.all(u[fixed] == 0.0)


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("variant,exchange", [(0, 0), (0, 1), (1, 0), (1, 1)],
                         ids=["std-allgather", "std-halo", "single-allgather", "single-halo"])
def test_loopback_overlap_matches_oracle_cfg3(lib, G, variant, exchange):
    """f1 overlap: the exchange of the search direction on a side stream while the interior chunks
    are multiplied, the boundary chunks after the join (fsfem_set_overlap)."""
    m = config_mesh(3)
    uo = np.load(os.path.join(GOLDEN, "oracle_cfg3_u.npy"))
    u, rep, rng = solve_group(lib, m, G, variant, exchange, overlap=True)
    assert rep["converged"] == 1 and rep["rel_residual"] <= 1e-10
    assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)
    u2, rep2, _ = solve_group(lib, m, G, variant, exchange, overlap=True)
    assert np.array_equal(u, u2)  # the side stream does not make the result timing dependent


def test_loopback_bitwise_reproducible(lib):
    m = config_mesh(3)
    u1, r1, _ = solve_group(lib, m, 3, 0, 1)
    u2, r2, _ = solve_group(lib, m, 3, 0, 1)
    assert np.array_equal(u1, u2) and r1["iterations"] == r2["iterations"]


def test_deterministic_dots_bit_identical_across_rank_counts(lib):
    """with deterministic dots the solve is bit-identical at G = 1, 2, 3, 4."""
    m = config_mesh(3)
    uo = np.load(os.path.join(GOLDEN, "oracle_cfg3_u.npy"))
    ref = None
    for G in (1, 2, 3, 4):
        for exchange in ((0,) if G == 1 else (0, 1)):
            u, rep, rng = solve_group(lib, m, G, 0, exchange, det=True)
            assert rep["converged"] == 1
            assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)
            if ref is None:
                ref = (u, rep["iterations"])
            else:
                assert rep["iterations"] == ref[1], (G, exchange)
                assert np.array_equal(u, ref[0]), (G, exchange, np.abs(u - ref[0]).max())


def test_loopback_ragged_and_permuted_mesh(lib):
    """Randomly relabelled ragged mesh: every rank's columns reach all others (no band)."""
    from oracle import Oracle
    m = kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8, tet_perm_seed=9)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    o.assemble_fs(E, NU)
    o.apply_bc(m.dirichlet, m.loads, 0)
    uo, _ = o.pcg(1e-10)
    for G, variant, exchange, det in ((2, 0, 1, False), (3, 1, 1, False), (3, 0, 0, True)):
        u, rep, _ = solve_group(lib, m, G, variant, exchange, det)
        assert rep["converged"] == 1
        assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo), (G, variant, exchange, det)


def test_loopback_errors(lib):
    import torch
    P = lib
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a, b = P.FsFem(stream=s1.cuda_stream), P.FsFem(stream=s2.cuda_stream)
    with pytest.raises(P.FsfemError) as e:
        P.fsfem_comm_init_loopback([a.ctx, b.ctx])  # different streams
    assert e.value.status == "INVALID_ARG"
    with pytest.raises(P.FsfemError) as e:
        P.fsfem_comm_init_loopback([a.ctx, a.ctx])
    assert e.value.status == "INVALID_ARG"
    m = config_mesh(1)
    a.build_faces(m.xyz, m.tets)
    with pytest.raises(P.FsfemError) as e:
        a.set_deterministic(True)  # after build_faces
    assert e.value.status == "STATE"
    a.close()
    b.close()
