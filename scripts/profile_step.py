#!/usr/bin/env python
"""One short pass of the hot path for ncu: faces, assembly (symbolic + numeric, then `--reassemble`
numeric-only repeats), BCs and a PCG bounded to `--pcg-iters` iterations (NOT_CONVERGED is fine).

    python scripts/profile_step.py --config 4 --pcg-iters 64 --reassemble 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--pcg-iters", type=int, default=64)
    ap.add_argument("--reassemble", type=int, default=2)
    ap.add_argument("--reorder", type=int, default=0, help="0 auto, 1 always, 2 never")
    ap.add_argument("--pcg-variant", type=int, default=0, help="0 standard, 1 single reduction")
    ap.add_argument("--loop", type=int, default=1, help="0 device while loop, 1 host-polled batches (default)")
    ap.add_argument("--solves", type=int, default=1, help="repeat the solve (steady-state timing)")
    ap.add_argument("--rebuild", type=int, default=0, help="extra faces + symbolic passes (steady-state timing)")
    a = ap.parse_args()
    import torch
    from fsfem_inputs import config_mesh
    from paper_2001_08849_b200 import FsFem, fsfem_apply_bc, fsfem_assemble_csr, fsfem_build_faces, fsfem_pcg_solve
    m = config_mesh(a.config)
    dev = torch.device("cuda", 0)
    g = FsFem(device=0, stream=torch.cuda.current_stream().cuda_stream)
    g.set_reorder(a.reorder)
    g.set_pcg_variant(a.pcg_variant)
    g.set_loop(a.loop)
    xyz = torch.from_numpy(m.xyz).to(dev)
    tets = torch.from_numpy(m.tets).to(dev)
    dirichlet = torch.from_numpy(m.dirichlet).to(dev)
    loads = torch.from_numpy(m.loads.reshape(-1).copy()).to(dev)
    u = torch.zeros(3 * m.n_nodes, dtype=torch.float64, device=dev)
    for _ in range(a.rebuild):
        fsfem_build_faces(g.ctx, xyz, tets)
        fsfem_assemble_csr(g.ctx, 1.0e6, 0.3)
        r = g.report()
        print(f"rebuild: faces {r['t_faces_ms']:.3f} ms, symbolic {r['t_symbolic_ms']:.3f} ms")
    fsfem_build_faces(g.ctx, xyz, tets)
    t_num = []
    for _ in range(1 + a.reassemble):
        fsfem_assemble_csr(g.ctx, 1.0e6, 0.3)
        t_num.append(round(g.report()["t_numeric_ms"], 4))
    print("numeric assembly ms per call:", t_num, "aux bytes", g.report()["assembly_aux_bytes"],
          "alg bytes", g.report()["assembly_bytes"])
    for _ in range(a.solves - 1):
        fsfem_assemble_csr(g.ctx, 1.0e6, 0.3)
        fsfem_apply_bc(g.ctx, dirichlet, loads, 0)
        try:
            r = fsfem_pcg_solve(g.ctx, u, True, 1e-10, a.pcg_iters, allow_not_converged=True)
        except Exception as e:  # tuning builds that skip work may break PCG: report the timings anyway
            r = g.report()
            print("solve error:", str(e)[:80])
        print(f"solve: {r['iterations']} it, {r['t_pcg_ms']:.3f} ms, {r['iterations'] / r['t_pcg_ms'] * 1e3:.0f} it/s, "
              f"spmv {r['t_spmv_ms'] / max(1, r['spmv_launches']) * 1e3:.2f} us (events), "
              f"{r['t_spmv_dev_ms'] / max(1, r['spmv_dev_launches']) * 1e3:.2f} us (device timer)")
    if a.solves > 1:
        fsfem_assemble_csr(g.ctx, 1.0e6, 0.3)
    fsfem_apply_bc(g.ctx, dirichlet, loads, 0)
    try:
        rep = fsfem_pcg_solve(g.ctx, u, True, 1e-10, a.pcg_iters, allow_not_converged=True)
    except Exception as e:  # tuning builds that skip work break PCG: report the timings anyway
        rep = g.report()
        rep["status"] = str(e)[:60]
    torch.cuda.synchronize()
    print({k: rep[k] for k in ("iterations", "status", "t_numeric_ms", "t_pcg_ms", "t_spmv_ms", "spmv_launches",
                               "reordered", "t_faces_ms", "t_symbolic_ms")})


if __name__ == "__main__":
    main()
