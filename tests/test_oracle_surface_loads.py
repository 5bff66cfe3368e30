"""Pins of oracle O10, the consistent nodal loads of a uniform surface traction (PAPER.md:449,
496-499 §4.1): total force = traction x loaded area (closed form), loads only on the loaded
surface's nodes, and linearity in the traction."""
import numpy as np

from fsfem_inputs import kuhn_beam
from oracle import Oracle


def test_top_face_pressure_totals():
    L, W, H = 1.0, 0.2, 0.2
    m = kuhn_beam(8, 3, 3, L=L, W=W, H=H, jitter=0.2, jitter_seed=2)  # jitter keeps the box faces flat
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    top = np.isclose(m.xyz[:, 2], H)
    p = 12500.0
    f = o.surface_loads(top, [0.0, 0.0, -p])
    assert np.isclose(f[:, 2].sum(), -p * L * W, rtol=1e-12)
    assert np.abs(f[:, :2]).max() == 0.0
    assert np.all(f[~top] == 0.0) and np.all(f[top, 2] < 0.0)
    # corner nodes of a Kuhn top face carry less than interior ones; all loads are p*A/3 sums
    f2 = o.surface_loads(top, [1.0, 2.0, 3.0])
    assert np.allclose(f2[:, 0] * -p, f[:, 2] * 1.0, rtol=1e-12)
    assert np.allclose(f2[:, 2], 3 * f2[:, 0], rtol=1e-12)


def test_whole_boundary_of_a_box_sums_to_zero_for_pressure_normal_free_load():
    """Every exterior face flagged: a constant traction vector integrates to t x total surface area."""
    m = kuhn_beam(3, 2, 2, L=2.0, W=1.0, H=1.0)
    o = Oracle(m.xyz, m.tets)
    o.build_faces()
    f = o.surface_loads(np.ones(m.n_nodes, bool), [0.0, 1.0, 0.0])
    area = 2 * (2.0 * 1.0 + 2.0 * 1.0 + 1.0 * 1.0)
    assert np.isclose(f[:, 1].sum(), area, rtol=1e-12)
