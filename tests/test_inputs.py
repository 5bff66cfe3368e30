"""Seeded input generator (fsfem_inputs): counts, determinism, jitter/permutation recipe."""
import numpy as np
import pytest

from fsfem_inputs import CONFIGS, config_mesh, kuhn_beam, kuhn_counts, splitmix64_stream, uniform01


def test_splitmix64_reference_values():
    # Published SplitMix64 (Steele, Lea, Flood 2014) outputs for seed 0 and seed 1234567.
    z = splitmix64_stream(0, 3)
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    z = splitmix64_stream(1234567, 2)
    assert [int(v) for v in z] == [6457827717110365317, 3203168211198807973]
    u = uniform01(splitmix64_stream(7, 100000))
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01


def test_stream_offsets_are_counter_based():
    a = splitmix64_stream(42, 10)
    b = splitmix64_stream(42, 4, start=6)
    assert np.array_equal(a[6:], b)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_config_counts(cfg):
    m = config_mesh(cfg)
    c = kuhn_counts(*m.grid)
    assert m.n_nodes == c["n_nodes"] and m.n_tets == c["n_tets"]
    nx, ny, nz = m.grid
    assert len(m.dirichlet) == (ny + 1) * (nz + 1) == len(m.tip)
    assert np.isclose(m.loads[:, 2].sum(), -1.0) and np.all(m.loads[:, :2] == 0)
    assert m.tets.dtype == np.int32 and m.tets.min() == 0 and m.tets.max() == m.n_nodes - 1


def test_baseline_node_counts():
    # cfg5 has 401*65*65 = 1,694,225 nodes (BASELINE.json's 1,690,065 is a slip).
    assert kuhn_counts(400, 64, 64)["n_nodes"] == 1_694_225
    assert kuhn_counts(200, 40, 40)["n_tets"] == 1_920_000
    assert kuhn_counts(200, 40, 40)["n_faces"] == 3_875_200
    assert kuhn_counts(200, 40, 40)["nnz_fs"] == 78_876_369


def _signed_vol(xyz, tets):
    p = xyz[tets]
    return np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0])) / 6.0


@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_all_tets_positive(cfg):
    m = config_mesh(cfg)
    v = _signed_vol(m.xyz, m.tets)
    assert v.min() > 0.0
    assert np.isclose(v.sum(), 10.0, rtol=1e-12)


def test_jitter_only_interior_and_bounded():
    a = config_mesh(3)
    b = kuhn_beam(100, 20, 20)
    d = a.xyz - b.xyz
    moved = np.any(d != 0, axis=1)
    nx, ny, nz = a.grid
    i = np.arange(a.n_nodes) % (nx + 1)
    j = (np.arange(a.n_nodes) // (nx + 1)) % (ny + 1)
    k = np.arange(a.n_nodes) // ((nx + 1) * (ny + 1))
    interior = (i > 0) & (i < nx) & (j > 0) & (j < ny) & (k > 0) & (k < nz)
    assert np.array_equal(moved, interior)
    h = np.array([10.0 / nx, 1.0 / ny, 1.0 / nz])
    assert np.all(np.abs(d) <= 0.15 * h + 1e-15)


def test_permutation_is_relabel():
    a = kuhn_beam(6, 3, 2, jitter=0.1, jitter_seed=9)
    b = kuhn_beam(6, 3, 2, jitter=0.1, jitter_seed=9, node_perm_seed=105, tet_perm_seed=205)
    # same multiset of tets (as coordinate sets), same clamped / tip coordinates
    ka = {tuple(sorted(map(tuple, a.xyz[t].round(12)))) for t in a.tets}
    kb = {tuple(sorted(map(tuple, b.xyz[t].round(12)))) for t in b.tets}
    assert ka == kb
    assert np.allclose(np.sort(a.xyz[a.dirichlet], axis=0), np.sort(b.xyz[b.dirichlet], axis=0))
    assert np.all(b.xyz[b.dirichlet, 0] == 0.0) and np.all(b.xyz[b.tip, 0] == 10.0)
    assert np.isclose(b.loads[b.tip, 2].sum(), -1.0)
    # deterministic
    c = kuhn_beam(6, 3, 2, jitter=0.1, jitter_seed=9, node_perm_seed=105, tet_perm_seed=205)
    assert np.array_equal(b.tets, c.tets) and np.array_equal(b.xyz, c.xyz)


def test_cfg5_shape():
    c = CONFIGS[5]
    assert c["grid"] == (400, 64, 64) and c["jitter"] == 0.2
