#!/usr/bin/env python
"""PCG iterations/s per loop mode (host batches, cluster kernel) on small configs.
Usage: [FSFEM_LIB=...] python scripts/loop_bench.py --configs 1 2 3"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--modes", type=int, nargs="+", default=[1, 2])
    a = ap.parse_args()
    from fsfem_inputs import config_mesh
    from paper_2001_08849_b200 import FsFem
    for cfg in a.configs:
        m = config_mesh(cfg)
        for mode in a.modes:
            g = FsFem()
            g.set_loop(mode)
            g.build_faces(m.xyz, m.tets)
            g.assemble_csr(1.0e6, 0.3)
            g.apply_bc(m.dirichlet, m.loads.reshape(-1))
            best = None
            for _ in range(3):
                u, rep = g.pcg_solve(rel_tol=1e-10)
                t = rep["t_pcg_ms"] / max(rep["iterations"], 1) * 1e3
                best = t if best is None else min(best, t)
            print(f"cfg{cfg} loop {rep['pcg_loop']} (asked {mode}): {rep['iterations']} it, {best:.2f} us/it, "
                  f"{1e6 / best:.0f} it/s", flush=True)
            g.close()


if __name__ == "__main__":
    main()
