"""Halo of the row partition (fsfem_get_halo, fsfem_set_exchange).

The halo-only exchange sends each rank just the entries of p its rows read.  On one GPU the
exchange itself (NCCL send/recv) cannot run, so this checks what it relies on, per rank of
partition-only contexts: the halo equals the columns of the rank's CSR rows outside its range,
and the rank's SpMV rows computed from own + halo entries only (every other entry NaN) are
bitwise those computed from the full vector, for the SpMV kernel the mesh uses and both
large-mesh kernels.  The send/recv protocol is covered on CPU by tests/test_multirank_cpu.py."""
import os
import subprocess
import sys

import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam

pytestmark = pytest.mark.gpu

E, NU = 1.0e6, 0.3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2001_08849_b200 import FsFem, load_library
    load_library()
    return FsFem


def _check(fs, m, nranks):
    x = np.random.default_rng(nranks).standard_normal(3 * m.n_nodes)
    for r in range(nranks):
        g = fs()
        g.comm_init(None, r, nranks)
        g.set_exchange(1)
        g.build_faces(m.xyz, m.tets)
        rng = g.partition()
        lo, hi = int(rng[r]), int(rng[r + 1])
        g.assemble_csr(E, NU)
        halo = g.halo()
        cols = np.unique(g.get_csr().col_idx // 3)
        want = cols[(cols < lo) | (cols >= hi)]
        assert np.array_equal(halo, want)
        assert np.all(np.diff(halo) > 0)
        xm = np.full_like(x, np.nan)
        keep = np.concatenate([np.arange(lo, hi), halo])
        for a in range(3):
            xm[3 * keep + a] = x[3 * keep + a]
        q_full = g.spmv(x)[3 * lo:3 * hi]
        q_halo = g.spmv(xm)[3 * lo:3 * hi]
        assert np.all(np.isfinite(q_halo))
        assert np.array_equal(q_halo, q_full)


@pytest.mark.parametrize("nranks", [2, 3])
def test_halo_small_mesh(fs, nranks):
    _check(fs, kuhn_beam(9, 5, 3, L=4.0, jitter=0.25, jitter_seed=4, node_perm_seed=8, tet_perm_seed=9), nranks)


_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import test_gpu_halo as t
from fsfem_inputs import config_mesh
from paper_2001_08849_b200 import FsFem, load_library
load_library()
t._check(FsFem, config_mesh(3), {nranks})
print("ok")
"""


@pytest.mark.parametrize("kernel", ["gather", "dataflow"])
def test_halo_cfg3_large_kernels(kernel):
    env = dict(os.environ, FSFEM_SPMV_KERNEL=kernel)
    out = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), nranks=2)],
                         env=env, check=True, timeout=600, capture_output=True, text=True)
    assert out.stdout.strip().endswith("ok")


def test_exchange_mode_errors(fs):
    from paper_2001_08849_b200 import FsfemError
    m = config_mesh(1)
    g = fs()
    with pytest.raises(FsfemError) as e:
        g.set_exchange(5)
    assert e.value.status == "INVALID_ARG"
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    assert g.halo().size == 0  # one rank: no halo
    with pytest.raises(FsfemError) as e:
        g.set_exchange(1)
    assert e.value.status == "STATE"
