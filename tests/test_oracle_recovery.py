"""Pins of the oracle's strain/stress recovery O9 against
what the mathematics fixes: rigid motions carry no strain, a linear displacement field has the
constant strain sym(grad u) in every smoothing domain (FS-FEM is linearly exact), isotropic
Hooke's law in Lame form, and the nodal average of a constant field is that field."""
import numpy as np
import pytest

from fsfem_inputs import kuhn_beam
from oracle import Oracle


def _mesh():
    return kuhn_beam(3, 2, 2, L=2.0, jitter=0.2, jitter_seed=21)


def _voigt_from_grad(G):
    """Engineering-shear Voigt strain (xx, yy, zz, yz, xz, xy) of displacement gradient G[i][j] = du_i/dx_j."""
    return np.array([G[0, 0], G[1, 1], G[2, 2], G[1, 2] + G[2, 1], G[0, 2] + G[2, 0], G[0, 1] + G[1, 0]])


def _hooke(E, nu, eps):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    tr = eps[0] + eps[1] + eps[2]
    return np.array([lam * tr + 2 * mu * eps[0], lam * tr + 2 * mu * eps[1], lam * tr + 2 * mu * eps[2],
                     mu * eps[3], mu * eps[4], mu * eps[5]])


def test_zero_and_rigid_motions_have_no_strain():
    m = _mesh()
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    for u in (np.zeros_like(m.xyz), np.tile([0.3, -0.2, 0.7], (m.n_nodes, 1)),
              np.cross(np.array([0.01, -0.02, 0.015]), m.xyz - m.xyz.mean(0))):
        eps, sig, ns, vm = o.recover(1.0e6, 0.3, u)
        assert np.abs(eps).max() <= 1e-13 * max(1.0, np.abs(u).max())
        assert np.abs(vm).max() <= 1e-13 * 1.0e6 * max(1.0, np.abs(u).max())


def test_linear_field_gives_exact_constant_strain_and_stress():
    m = _mesh()
    o = Oracle(m.xyz, m.tets)
    nf, _ = o.build_faces()[0].shape
    rng = np.random.default_rng(5)
    G = rng.standard_normal((3, 3)) * 1e-3
    u = m.xyz @ G.T + np.array([0.1, 0.2, -0.3])
    E, nu = 2.0e8, 0.3
    eps, sig, ns, vm = o.recover(E, nu, u)
    e_ref = _voigt_from_grad(G)
    s_ref = _hooke(E, nu, e_ref)
    assert eps.shape == (nf, 6)
    assert np.abs(eps - e_ref).max() <= 1e-10 * np.abs(e_ref).max()
    assert np.abs(sig - s_ref).max() <= 1e-10 * np.abs(s_ref).max()
    # constant field: every nodal average equals it
    assert np.abs(ns - s_ref).max() <= 1e-10 * np.abs(s_ref).max()
    d = s_ref
    vm_ref = np.sqrt(0.5 * ((d[0] - d[1]) ** 2 + (d[1] - d[2]) ** 2 + (d[2] - d[0]) ** 2) + 3 * (d[3:] ** 2).sum())
    assert np.allclose(vm, vm_ref, rtol=1e-10)


def test_uniaxial_and_hydrostatic():
    m = _mesh()
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    u = np.zeros_like(m.xyz)
    u[:, 0] = 0.001 * m.xyz[:, 0]
    eps, sig, ns, vm = o.recover(1.0e6, 0.0, u)  # nu = 0: sigma_xx = E eps_xx, the rest zero
    assert np.allclose(sig, [1000.0, 0, 0, 0, 0, 0], atol=1e-9)
    assert np.allclose(vm, 1000.0, rtol=1e-12)
    eps, sig, ns, vm = o.recover(1.0e6, 0.3, 0.002 * (m.xyz - 1.0))  # pure dilatation
    assert np.abs(vm).max() <= 1e-9 * np.abs(ns).max()
