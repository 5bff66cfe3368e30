"""Offline: run the CPU ORACLE alone on a full BASELINE config and record reference values.

Writes tests/golden/oracle_cfg<N>.json: faces, nnz, PCG iterations, residuals, tip deflection
and a deterministic sample of displacement entries.  Calls only oracle/ and fsfem_inputs/
(never the CUDA path).  Used by tests (parity at full size) and by bench.py's CPU baseline
(iteration count of the full solve).  Usage: python scripts/oracle_full_solve.py 4 [chunks] [--fem] [--u-only]
--u-only: write only tests/golden/oracle_cfg<N>_u.npy (the whole displacement vector; any config).
--fem: the oracle's FEM-T4 companion (O8) instead of FS-FEM ->
tests/golden/oracle_cfg<N>_fem.json (the FS >= FEM tip-deflection pin).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from fsfem_inputs import config_mesh  # noqa: E402
from oracle import Oracle  # noqa: E402

E, NU = 1.0e6, 0.3


def main(cfg: int, chunks: int = 4, fem: bool = False, u_only: bool = False):
    m = config_mesh(cfg)
    o = Oracle(m.xyz, m.tets)
    t = {}
    t0 = time.perf_counter()
    o.build_faces()
    t["faces_s"] = time.perf_counter() - t0
    bounds = np.linspace(0, m.n_nodes, chunks + 1).astype(int)
    rps, cis, vas = [], [], []
    off = 0
    t0 = time.perf_counter()
    for a, b in zip(bounds[:-1], bounds[1:]):
        lo, rp, ci, va = (o.assemble_fem if fem else o.assemble_fs)(E, NU, int(a), int(b))
        rps.append(rp[:-1] + off)
        off += rp[-1]
        cis.append(ci)
        vas.append(va)
        print(f"rows {a}..{b} assembled at {time.perf_counter() - t0:.1f}s", flush=True)
    t["assemble_s"] = time.perf_counter() - t0
    rp = np.concatenate(rps + [np.array([off])])
    ci = np.concatenate(cis)
    va = np.concatenate(vas)
    del rps, cis, vas
    o.set_csr(rp, ci, va)
    t0 = time.perf_counter()
    o.apply_bc(m.dirichlet, m.loads, 0)
    t["bc_s"] = time.perf_counter() - t0
    u, rep = o.pcg(1e-10)
    t["pcg_s"] = o.timings["pcg_s"]
    rng = np.random.default_rng(12345)
    idx = np.sort(rng.choice(u.size, 4096, replace=False))
    out = dict(config=cfg, n_nodes=m.n_nodes, n_tets=m.n_tets, n_faces=o.n_faces, n_interior=o.n_interior,
               nnz=int(rp[-1]), pcg=rep, tip_mean_uz=float(u.reshape(-1, 3)[m.tip, 2].mean()),
               u_norm=float(np.linalg.norm(u)), u_sample_idx=idx.tolist(), u_sample=u[idx].tolist(),
               f_dot_u=float(m.loads.reshape(-1) @ u), timings_s=t, threads=int(os.environ.get("OMP_NUM_THREADS", "0")),
               method="FEM-T4" if fem else "FS-FEM",
               note="written by scripts/oracle_full_solve.py from oracle/ only")
    path = os.path.join(ROOT, "tests", "golden", f"oracle_cfg{cfg}{'_fem' if fem else ''}.json")
    if not u_only:
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
    if (cfg <= 4 or u_only) and not fem:
        np.save(os.path.join(ROOT, "tests", "golden", f"oracle_cfg{cfg}_u.npy"), u)
    print(json.dumps({k: v for k, v in out.items() if not k.startswith("u_sample")}, indent=1))


if __name__ == "__main__":
    pos = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(int(pos[0]), int(pos[1]) if len(pos) > 1 else 4, fem="--fem" in sys.argv, u_only="--u-only" in sys.argv)
