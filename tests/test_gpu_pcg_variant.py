"""Single-reduction PCG (fsfem_set_pcg_variant, Chronopoulos-Gear form of the same Jacobi-PCG;
SURVEY.md 8(f) f1) against the oracle's standard PCG: same solution to the parity bar, iteration
counts within 5%, bitwise reproducible, and the variant switch back to the standard form."""
import json
import os

import numpy as np
import pytest

from fsfem_inputs import config_mesh, kuhn_beam
from oracle import Oracle

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


def _solve(fs, m, variant):
    g = fs()
    g.set_pcg_variant(variant)
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve(rel_tol=1e-10)
    return g, u, rep


@pytest.mark.parametrize("name,m", [("cfg2", config_mesh(2)),
                                    ("ragged", kuhn_beam(7, 3, 5, L=3.0, jitter=0.2, jitter_seed=17))])
def test_single_reduction_matches_oracle(fs, name, m):
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    o.assemble_fs(E, NU)
    o.apply_bc(m.dirichlet, m.loads, 0)
    u_ref, orep = o.pcg(1e-10)
    _, u, rep = _solve(fs, m, 1)
    assert rep["converged"] == 1 and rep["rel_residual"] <= 1e-10
    assert rep["true_rel_residual"] < 1e-8
    assert np.linalg.norm(u - u_ref) <= 1e-7 * np.linalg.norm(u_ref)
    assert abs(rep["iterations"] - orep["iterations"]) <= max(3, 0.05 * orep["iterations"])


def test_single_reduction_cfg3_and_reproducible(fs):
    m = config_mesh(3)
    uo = np.load(os.path.join(ROOT, "tests", "golden", "oracle_cfg3_u.npy"))
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_cfg3.json")))
    _, u1, r1 = _solve(fs, m, 1)
    _, u2, r2 = _solve(fs, m, 1)
    assert np.linalg.norm(u1 - uo) <= 1e-7 * np.linalg.norm(uo)
    assert abs(r1["iterations"] - gold["pcg"]["iterations"]) <= 0.05 * gold["pcg"]["iterations"]
    assert np.array_equal(u1, u2) and r1["iterations"] == r2["iterations"]


def test_single_reduction_cfg4_dataflow_spmv(fs):
    """cfg4 runs the dataflow SpMV; its last CTA also reduces the update kernel's partials."""
    m = config_mesh(4)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_cfg4.json")))
    g, u, rep = _solve(fs, m, 1)
    assert rep["converged"] == 1 and rep["spmv_kernel"] == 2
    f = m.loads.reshape(-1)
    assert abs(f @ u - gold["f_dot_u"]) <= 1e-8 * abs(gold["f_dot_u"])
    idx = np.asarray(gold["u_sample_idx"])
    assert np.abs(u[idx] - np.asarray(gold["u_sample"])).max() <= 1e-7 * gold["u_norm"]


def test_variant_switch_and_errors(fs):
    from paper_2001_08849_b200 import FsfemError
    m = config_mesh(1)
    g = fs()
    with pytest.raises(FsfemError) as e:
        g.set_pcg_variant(3)
    assert e.value.status == "INVALID_ARG"
    g.build_faces(m.xyz, m.tets)
    g.assemble_csr(E, NU)
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    g.set_pcg_variant(1)
    u1, r1 = g.pcg_solve()
    g.set_pcg_variant(0)
    u0, r0 = g.pcg_solve()
    assert np.linalg.norm(u1 - u0) <= 1e-8 * np.linalg.norm(u0)
    g.set_pcg_variant(2)  # auto: standard on one GPU
    u2, r2 = g.pcg_solve()
    assert np.array_equal(u2, u0) and r2["iterations"] == r0["iterations"]
