"""World-size-2 (and 3) CPU run of the multi-GPU row partition over `gloo`.

The library's N>1 path (api.cu: fsfem_comm_init, pcg_iteration, combine, gather_full) needs one
GPU per rank, which this container and the round's GPU box do not have.  This test runs the same
host-side protocol with torch.distributed/gloo between CPU processes, each rank holding only its
rows (assembled by the oracle for its node range), and checks it against the single-process
oracle solve:
  * partition: rank r owns nodes [r*ceil(N/G), min(N, (r+1)*ceil(N/G))) (include/fsfem.h);
  * BCs (MODIFY) applied on own rows with the global clamp mask (bc.cu);
  * per iteration: all_gather of equal padded p slices (ncclAllGather in gather_full), dot
    partials all_gathered and summed in rank order (combine), the same recurrence as pcg.cuh;
  * the single-reduction variant (fsfem_set_pcg_variant): one combined all_gather of
    (u.w, r.u, r.r) per iteration (k_combine stage 4);
  * the halo exchange (fsfem_set_exchange): only the halo entries of p are sent / received
    (remote entries outside the halo are NaN and must never be read).
The GPU side of the partition (halo blocks, transposed lists, per-rank CSR/SpMV/BC rows) is
covered by tests/test_gpu_parity.py::test_row_partition_contexts.
"""
import os
import socket

import numpy as np
import pytest

E, NU = 1.0e6, 0.3


def _mesh():
    from fsfem_inputs import kuhn_beam
    return kuhn_beam(9, 3, 3, L=4.0, jitter=0.2, jitter_seed=11, node_perm_seed=12, tet_perm_seed=13)


def _partition(nn, nranks, r):
    chunk = -(-nn // nranks)
    lo = min(nn, r * chunk)
    return lo, min(nn, lo + chunk), chunk


def _worker(rank, world, port, out_dir, variant="standard", exchange="allgather"):
    import torch
    import torch.distributed as dist
    from oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = _mesh()
    nn = m.n_nodes
    lo, hi, chunk = _partition(nn, world, rank)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    _, rp, ci, va = o.assemble_fs(E, NU, lo, hi)  # own rows, global columns
    va = va.copy()
    fixed = np.zeros(nn, bool)
    fixed[m.dirichlet] = True
    nrow = 3 * (hi - lo)
    diag = np.zeros(nrow)
    for k in range(nrow):
        r = 3 * lo + k
        for e in range(rp[k], rp[k + 1]):
            c = ci[e]
            if (fixed[r // 3] or fixed[c // 3]) and c != r:
                va[e] = 0.0
            if c == r:
                diag[k] = va[e]
    f = m.loads.reshape(-1)[3 * lo:3 * hi].copy()
    f[np.repeat(fixed[lo:hi], 3)] = 0.0
    dinv = 1.0 / diag

    def spmv(p_full):
        q = np.zeros(nrow)
        for k in range(nrow):
            s = 0.0
            for e in range(rp[k], rp[k + 1]):
                s += va[e] * p_full[ci[e]]
            q[k] = s
        return q

    def allgather_full(v_own):
        buf = torch.zeros(3 * chunk, dtype=torch.float64)
        buf[:nrow] = torch.from_numpy(v_own)
        parts = [torch.zeros(3 * chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, buf)
        return torch.cat(parts).numpy()[:3 * nn]

    # halo exchange (api.cu setup_halo / halo_exchange): the halo = columns of the own rows
    # outside the range, ascending; counts all-gathered, then each rank sends every owner the
    # list of that owner's nodes it needs; per exchange: send the needed entries, receive the halo
    cols = np.unique(ci // 3)
    halo = cols[(cols < lo) | (cols >= hi)]
    owner = np.minimum(halo // chunk, world - 1)
    need = np.array([np.sum(owner == q) for q in range(world)], np.int64)
    allneed = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allneed, torch.from_numpy(need))
    send_cnt = [int(allneed[q][rank]) if q != rank else 0 for q in range(world)]
    send_nodes = {}
    for q in range(world):  # pairwise, in rank order on both sides (no deadlock with gloo)
        if q == rank:
            continue
        lst = torch.from_numpy(halo[owner == q].astype(np.int64))
        got = torch.zeros(send_cnt[q], dtype=torch.int64)
        if rank < q:
            if lst.numel():
                dist.send(lst, q)
            if got.numel():
                dist.recv(got, q)
        else:
            if got.numel():
                dist.recv(got, q)
            if lst.numel():
                dist.send(lst, q)
        send_nodes[q] = got.numpy()
    full_p = np.full(3 * nn, np.nan)  # remote entries outside the halo stay NaN: never read

    def halo_full(v_own):
        full_p[3 * lo:3 * hi] = v_own
        for q in range(world):
            if q == rank:
                continue
            sbuf = torch.from_numpy(np.stack([full_p[3 * send_nodes[q] + a] for a in range(3)], 1).reshape(-1).copy())
            rn = halo[owner == q]
            rbuf = torch.zeros(3 * rn.size, dtype=torch.float64)
            if rank < q:
                if sbuf.numel():
                    dist.send(sbuf, q)
                if rbuf.numel():
                    dist.recv(rbuf, q)
            else:
                if rbuf.numel():
                    dist.recv(rbuf, q)
                if sbuf.numel():
                    dist.send(sbuf, q)
            rb = rbuf.numpy().reshape(-1, 3)
            for a in range(3):
                full_p[3 * rn + a] = rb[:, a]
        return full_p.copy()

    def gather_full(v_own):
        return halo_full(v_own) if exchange == "halo" else allgather_full(v_own)

    def combine(*vals):
        mine = torch.tensor(vals, dtype=torch.float64)
        parts = [torch.zeros(len(vals), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, mine)
        tot = np.zeros(len(vals))
        for p in parts:  # rank order
            tot += p.numpy()
        return tot

    x = np.zeros(nrow)
    r = f.copy()
    z = dinv * r
    p = z.copy()
    rho, rr, ff = combine(r @ z, r @ r, f @ f)
    it = 0
    tol = 1e-10
    if variant == "single_reduction":
        # Chronopoulos-Gear (pcg.cuh finish_cg, api.cu pcg_iteration_cg): ONE combined collective
        # of (u.w, r.u, r.r) per iteration; u = D^-1 r gathered, w = K u on own rows
        u = z
        w = spmv(gather_full(u))
        (delta,) = combine(u @ w)
        gamma = rho
        alpha = gamma / delta
        beta = 0.0
        alpha_prev = alpha
        ps = np.zeros(nrow)
        ss = np.zeros(nrow)
        while True:
            ps = u + beta * ps
            ss = w + beta * ss
            x += alpha * ps
            r -= alpha * ss
            u = dinv * r
            w = spmv(gather_full(u))
            delta, gamma_new, rr = combine(u @ w, r @ u, r @ r)
            it += 1
            if np.sqrt(rr) <= tol * np.sqrt(ff) or it >= 5000:
                break
            beta = gamma_new / gamma
            alpha = gamma_new / (delta - beta * gamma_new / alpha_prev)
            alpha_prev = alpha
            gamma = gamma_new
    while variant == "standard" and np.sqrt(rr) > tol * np.sqrt(ff) and it < 5000:
        q = spmv(gather_full(p))
        (pq,) = combine(p @ q)
        alpha = rho / pq
        x += alpha * p
        r -= alpha * q
        z = dinv * r
        rr, rz = combine(r @ r, r @ z)
        it += 1
        if np.sqrt(rr) <= tol * np.sqrt(ff):
            break
        beta = rz / rho
        rho = rz
        p = z + beta * p
    u = allgather_full(x)
    np.save(os.path.join(out_dir, f"u{rank}.npy"), u)
    np.save(os.path.join(out_dir, f"it{rank}.npy"), np.array([it]))
    dist.destroy_process_group()


def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,variant,exchange", [(2, "standard", "allgather"), (3, "standard", "allgather"),
                                                    (2, "single_reduction", "allgather"),
                                                    (3, "single_reduction", "halo"), (3, "standard", "halo")])
def test_row_partition_pcg_over_gloo(tmp_path, world, variant, exchange):
    import torch.multiprocessing as mp
    from oracle import Oracle
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), variant, exchange), nprocs=world, join=True)
    m = _mesh()
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    o.assemble_fs(E, NU)
    o.apply_bc(m.dirichlet, m.loads, 0)
    u_ref, rep = o.pcg(1e-10)
    us = [np.load(tmp_path / f"u{r}.npy") for r in range(world)]
    its = [int(np.load(tmp_path / f"it{r}.npy")[0]) for r in range(world)]
    for u in us[1:]:
        assert np.array_equal(u, us[0])  # every rank ends with the same full solution
    assert len(set(its)) == 1
    assert np.linalg.norm(us[0] - u_ref) <= 1e-7 * np.linalg.norm(u_ref)
    assert abs(its[0] - rep["iterations"]) <= max(3, 0.05 * rep["iterations"])
    fixed = np.repeat(np.isin(np.arange(m.n_nodes), m.dirichlet), 3)
    assert np.all(us[0][fixed] == 0.0)
