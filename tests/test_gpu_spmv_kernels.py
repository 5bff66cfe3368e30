"""Both large-mesh SpMV kernels of pcg.cu against the oracle, whichever the library picks by default.

`k_spmv` (gather: K_ji read transposed from row j) and `k_spmv_df` (dataflow push: row i pushes
K_ij^T x_i, row j sums its slots once the producer chunks are done) are selected with
FSFEM_SPMV_KERNEL, read once per process, so each case runs in its own interpreter.  Checked:
K x against the oracle's CSR product (1e-12 relative to max|K x|), the cfg3 solve against the
oracle's full solve, and run-to-run bitwise equality (every sum has a fixed order in both).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from fsfem_inputs import config_mesh
from paper_2001_08849_b200 import FsFem, load_library
load_library()
m = config_mesh({cfg})
x = np.random.default_rng(7).standard_normal(3 * m.n_nodes)
outs = []
for _ in range(2):
    g = FsFem()
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(1.0e6, 0.3)
    y = g.spmv(x)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve(rel_tol=1e-10)
    outs.append((y, u, rep["iterations"]))
np.savez({out!r}, y0=outs[0][0], y1=outs[1][0], u0=outs[0][1], u1=outs[1][1],
         it=np.array([outs[0][2], outs[1][2]]))
"""


def _run(kernel, cfg, tmp_path):
    out = str(tmp_path / f"{kernel}_{cfg}.npz")
    env = dict(os.environ, FSFEM_SPMV_KERNEL=kernel)
    subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, cfg=cfg, out=out)], env=env, check=True,
                   timeout=600)
    return np.load(out)


@pytest.mark.parametrize("kernel", ["gather", "dataflow"])
def test_spmv_kernel_cfg3(kernel, tmp_path):
    from fsfem_inputs import config_mesh
    from oracle import Oracle
    r = _run(kernel, 3, tmp_path)
    m = config_mesh(3)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    o.assemble_fs(1.0e6, 0.3)
    x = np.random.default_rng(7).standard_normal(3 * m.n_nodes)
    y_ref = o.spmv(x)
    assert np.abs(r["y0"] - y_ref).max() <= 1e-12 * np.abs(y_ref).max()
    uo = np.load(os.path.join(ROOT, "tests", "golden", "oracle_cfg3_u.npy"))
    assert np.linalg.norm(r["u0"] - uo) <= 1e-7 * np.linalg.norm(uo)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_cfg3.json")))
    assert abs(int(r["it"][0]) - gold["pcg"]["iterations"]) <= 0.05 * gold["pcg"]["iterations"]
    # bitwise reproducible
    assert np.array_equal(r["y0"], r["y1"]) and np.array_equal(r["u0"], r["u1"]) and r["it"][0] == r["it"][1]


def test_gather_and_dataflow_agree_cfg4(tmp_path):
    """cfg4 (bench workload): the two kernels give the same K x to rounding (different, fixed
    summation orders) and solutions within the parity bar of each other."""
    a = _run("gather", 4, tmp_path)
    b = _run("dataflow", 4, tmp_path)
    assert np.abs(a["y0"] - b["y0"]).max() <= 1e-12 * np.abs(a["y0"]).max()
    assert np.linalg.norm(a["u0"] - b["u0"]) <= 1e-7 * np.linalg.norm(a["u0"])
    assert np.array_equal(b["y0"], b["y1"]) and np.array_equal(b["u0"], b["u1"])


_PART_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from fsfem_inputs import config_mesh
from paper_2001_08849_b200 import FsFem, load_library
load_library()
m = config_mesh(3)
x = np.random.default_rng(11).standard_normal(3 * m.n_nodes)
g = FsFem()
g.build_faces(m.xyz, m.tets)
g.assemble_csr(1.0e6, 0.3)
full = g.spmv(x)
res = {{"full": full}}
for nranks in (2, 3):
    for r in range(nranks):
        h = FsFem()
        h.comm_init(None, r, nranks)
        h.build_faces(m.xyz, m.tets)
        rng = h.partition()
        lo, hi = int(rng[r]), int(rng[r + 1])
        res[f"r{{nranks}}"] = rng
        h.assemble_csr(1.0e6, 0.3)
        res[f"q{{nranks}}_{{r}}"] = h.spmv(x)[3 * lo:3 * hi]
        res[f"k{{nranks}}_{{r}}"] = np.array([h.report()["spmv_kernel"]])
np.savez({out!r}, **res)
"""


@pytest.mark.parametrize("kernel", ["gather", "dataflow"])
def test_spmv_kernel_row_partition(kernel, tmp_path):
    """Partition-only contexts (2 and 3 ranks' rows on one GPU, halo columns below the rank's
    range stored in the rows): each rank's rows of K x equal the single-context product."""
    out = str(tmp_path / f"part_{kernel}.npz")
    env = dict(os.environ, FSFEM_SPMV_KERNEL=kernel)
    subprocess.run([sys.executable, "-c", _PART_SCRIPT.format(root=ROOT, out=out)], env=env, check=True, timeout=600)
    r = np.load(out)
    full = r["full"]
    n_nodes = full.size // 3
    want = 1 if kernel == "gather" else 2
    for nranks in (2, 3):
        rng = r[f"r{nranks}"]
        for k in range(nranks):
            lo, hi = int(rng[k]), int(rng[k + 1])
            q = r[f"q{nranks}_{k}"]
            assert np.abs(q - full[3 * lo:3 * hi]).max() <= 1e-12 * np.abs(full).max()
            assert int(r[f"k{nranks}_{k}"][0]) in (0, want)  # small partitions may fall back to warp per node
