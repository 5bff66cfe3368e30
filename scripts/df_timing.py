#!/usr/bin/env python
"""Per-warp clock accounting of the dataflow SpMV (tuning build with FSFEM_DF_TIMING=1):
    python -m paper_2001_08849_b200.build --out build/libfsfem_dft.so -DFSFEM_DF_TIMING=1
    FSFEM_LIB=build/libfsfem_dft.so python scripts/df_timing.py | grep -A40 "=== timed"
Each sampled CTA prints, per warp role, the cycles spent waiting (A), in fences / copies (B) and
working (C), and its end time (S8)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fsfem_inputs import config_mesh
from paper_2001_08849_b200 import FsFem, fsfem_spmv
m = config_mesh(4)
g = FsFem(device=0, stream=torch.cuda.current_stream().cuda_stream)
g.build_faces(m.xyz, m.tets)
g.assemble_csr(1.0e6, 0.3)
x = torch.randn(3 * m.n_nodes, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    fsfem_spmv(g.ctx, x, y)
torch.cuda.synchronize()
print("=== timed", flush=True)
fsfem_spmv(g.ctx, x, y)
torch.cuda.synchronize()
