#!/usr/bin/env python
"""Repeated fsfem_spmv on one config (tuning experiments; includes the API's x/y copies).
Usage: FSFEM_LIB=... python scripts/spmv_bench.py --config 4 --reps 200"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    import torch
    from fsfem_inputs import config_mesh
    from paper_2001_08849_b200 import FsFem, fsfem_spmv
    m = config_mesh(a.config)
    g = FsFem(device=0, stream=torch.cuda.current_stream().cuda_stream)
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(1.0e6, 0.3)
    x = torch.randn(3 * m.n_nodes, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(10):
        fsfem_spmv(g.ctx, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            fsfem_spmv(g.ctx, x, y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / a.reps * 1e3)
    ts.sort()
    print(f"spmv cfg{a.config}: {ts[0]:.1f} us min / {ts[2]:.1f} median per call (incl. 2 D2D vector copies), "
          f"kernel {g.report()['spmv_kernel']}")


if __name__ == "__main__":
    main()
