#!/usr/bin/env python
"""Cold-path phase times (faces, symbolic, tile build) on one config, repeated on one context as
bench.py's step does.  Usage: FSFEM_PHASE_TIMES=1 python scripts/cold_path.py --config 4 --reps 3"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    from fsfem_inputs import config_mesh
    from paper_2001_08849_b200 import FsFem, fsfem_assemble_csr, fsfem_build_faces
    m = config_mesh(a.config)
    stream = torch.cuda.Stream()
    g = FsFem(device=0, stream=stream.cuda_stream)
    xyz = torch.from_numpy(m.xyz).cuda()
    tets = torch.from_numpy(m.tets).cuda()
    torch.cuda.synchronize()
    for r in range(a.reps):
        print(f"--- rep {r}", file=sys.stderr, flush=True)
        fsfem_build_faces(g.ctx, xyz, tets)
        fsfem_assemble_csr(g.ctx, 1.0e6, 0.3)
        rep = g.report()
        print(f"rep {r}: faces {rep['t_faces_ms']:.3f} ms, symbolic {rep['t_symbolic_ms']:.3f} ms, "
              f"numeric {rep['t_numeric_ms']:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
