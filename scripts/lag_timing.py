#!/usr/bin/env python
"""Per-warp clock accounting of k_spmv_lag (tuning builds with -DFSFEM_LAG_TIMING=1).
Usage: FSFEM_LIB=build/libfsfem_lagT.so FSFEM_SPMV_KERNEL=lag python scripts/lag_timing.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from fsfem_inputs import config_mesh  # noqa: E402
from paper_2001_08849_b200 import FsFem  # noqa: E402

m = config_mesh(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
g = FsFem()
g.build_faces(m.xyz, m.tets)
g.assemble_csr(1.0e6, 0.3)
x = np.random.default_rng(1).standard_normal(3 * m.n_nodes)
for _ in range(3):
    g.spmv(x)
    sys.stdout.flush()
    print("-- call", flush=True)
