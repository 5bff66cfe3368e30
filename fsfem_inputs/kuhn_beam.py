"""Kuhn-tet cantilever beams (BASELINE.json configs[0..4]).

Stand-in for the paper's TetGen meshes of a cantilever (PAPER.md:496-559,
Table 3), which are not available: a box L x W x H split into nx*ny*nz hexes,
each hex cut into 6 tets sharing its main diagonal (Freudenthal/Kuhn split,
SURVEY.md Q18).  Nothing here evaluates the method; see DESIGN.md "Input recipe".

Conventions:
  * grid node (i,j,k) has id i + (nx+1)*(j + (ny+1)*k), x = i*L/nx, ...
  * hex h = i + nx*(j + ny*k) -> tets 6h..6h+5, one per axis permutation pi:
      [v0, v0+e_pi0, v0+e_pi0+e_pi1, v0+(1,1,1)]  with the last two swapped for
      odd pi, so every tet has a positive determinant before jitter.
  * jitter: interior nodes (0<i<nx, 0<j<ny, 0<k<nz) move by (2u-1)*J*h_axis,
      u = the (3*node+axis+1)-th output of SplitMix64 seeded with `jitter_seed`.
  * relabel: new node order = stable argsort of SplitMix64(node_perm_seed)
      outputs; tet order likewise with tet_perm_seed.  Vertex order inside a
      tet is kept.
  * clamped nodes = grid nodes with i == 0; tip nodes = i == nx, each carrying
      f_z = P / n_tip (P = -1).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# The six axis permutations, in the fixed order of SURVEY.md 8(d).
_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_ODD = (False, True, True, False, False, True)


def splitmix64_stream(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Outputs start+1 .. start+n of SplitMix64(seed) (counter form: s_k = seed + k*gamma)."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(z: np.ndarray) -> np.ndarray:
    """u = (z >> 11) * 2^-53 in [0, 1)."""
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


@dataclass
class BeamMesh:
    xyz: np.ndarray          # float64 [N_n, 3]
    tets: np.ndarray         # int32   [N_t, 4], 0-based
    dirichlet: np.ndarray    # int32   [n_d]   clamped node ids (all 3 dofs)
    loads: np.ndarray        # float64 [N_n, 3] nodal forces
    tip: np.ndarray          # int32   [n_tip] node ids at x = L
    grid: tuple              # (nx, ny, nz)
    dims: tuple              # (L, W, H)
    meta: dict = field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])


def kuhn_beam(nx: int, ny: int, nz: int, L: float = 10.0, W: float = 1.0, H: float = 1.0,
              jitter: float = 0.0, jitter_seed: int = 0, node_perm_seed: int | None = None,
              tet_perm_seed: int | None = None, P: float = -1.0) -> BeamMesh:
    if min(nx, ny, nz) < 1:
        raise ValueError("grid must have at least one hex per axis")
    n1x, n1y, n1z = nx + 1, ny + 1, nz + 1
    nn = n1x * n1y * n1z
    ii, jj, kk = np.meshgrid(np.arange(n1x), np.arange(n1y), np.arange(n1z), indexing="ij")
    # node id = i + n1x*(j + n1y*k): flatten in (k, j, i) order
    gi = ii.transpose(2, 1, 0).reshape(-1)
    gj = jj.transpose(2, 1, 0).reshape(-1)
    gk = kk.transpose(2, 1, 0).reshape(-1)
    hx, hy, hz = L / nx, W / ny, H / nz
    xyz = np.empty((nn, 3), dtype=np.float64)
    xyz[:, 0] = gi * L / nx
    xyz[:, 1] = gj * W / ny
    xyz[:, 2] = gk * H / nz
    if jitter > 0.0:
        u = uniform01(splitmix64_stream(jitter_seed, 3 * nn)).reshape(nn, 3)
        d = (2.0 * u - 1.0) * jitter * np.array([hx, hy, hz])
        interior = (gi > 0) & (gi < nx) & (gj > 0) & (gj < ny) & (gk > 0) & (gk < nz)
        xyz[interior] += d[interior]

    # hexes in id order h = i + nx*(j + ny*k)
    hi, hj, hk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    hi = hi.transpose(2, 1, 0).reshape(-1)
    hj = hj.transpose(2, 1, 0).reshape(-1)
    hk = hk.transpose(2, 1, 0).reshape(-1)
    nh = nx * ny * nz

    def nid(di, dj, dk):
        return (hi + di) + n1x * ((hj + dj) + n1y * (hk + dk))

    tets = np.empty((nh, 6, 4), dtype=np.int64)
    for p, (perm, odd) in enumerate(zip(_PERMS, _ODD)):
        e = [0, 0, 0]
        v = [nid(0, 0, 0)]
        for ax in perm[:2]:
            e[ax] += 1
            v.append(nid(*e))
        v.append(nid(1, 1, 1))
        if odd:
            v[2], v[3] = v[3], v[2]
        for q in range(4):
            tets[:, p, q] = v[q]
    tets = tets.reshape(-1, 4)

    dirichlet = np.nonzero(gi == 0)[0]
    tip = np.nonzero(gi == nx)[0]
    loads = np.zeros((nn, 3), dtype=np.float64)
    loads[tip, 2] = P / len(tip)

    if node_perm_seed is not None:
        perm = np.argsort(splitmix64_stream(node_perm_seed, nn), kind="stable")  # perm[new] = old
        new_of_old = np.empty(nn, dtype=np.int64)
        new_of_old[perm] = np.arange(nn)
        xyz = xyz[perm]
        loads = loads[perm]
        tets = new_of_old[tets]
        dirichlet = np.sort(new_of_old[dirichlet])
        tip = np.sort(new_of_old[tip])
    if tet_perm_seed is not None:
        tperm = np.argsort(splitmix64_stream(tet_perm_seed, tets.shape[0]), kind="stable")
        tets = tets[tperm]

    return BeamMesh(xyz=np.ascontiguousarray(xyz), tets=np.ascontiguousarray(tets.astype(np.int32)),
                    dirichlet=dirichlet.astype(np.int32), loads=np.ascontiguousarray(loads),
                    tip=tip.astype(np.int32), grid=(nx, ny, nz), dims=(L, W, H),
                    meta=dict(jitter=jitter, jitter_seed=jitter_seed, node_perm_seed=node_perm_seed,
                              tet_perm_seed=tet_perm_seed, P=P))


# BASELINE.json configs[0..4] (1-based names cfg1..cfg5), E = 1e6, nu = 0.3.
CONFIGS = {
    1: dict(grid=(10, 2, 2), jitter=0.0),
    2: dict(grid=(40, 8, 8), jitter=0.0),
    3: dict(grid=(100, 20, 20), jitter=0.15, jitter_seed=3),
    4: dict(grid=(200, 40, 40), jitter=0.0),
    5: dict(grid=(400, 64, 64), jitter=0.2, jitter_seed=5, node_perm_seed=105, tet_perm_seed=205),
}
E_MOD = 1.0e6
NU = 0.3


def config_mesh(cfg: int, x_cells: int | None = None) -> BeamMesh:
    """Mesh of BASELINE config `cfg` (1..5).  `x_cells` < nx keeps the first x_cells
    hex columns at the same spacing (a slab of the same workload, used as the
    bounded CPU-oracle sample)."""
    c = CONFIGS[cfg]
    nx, ny, nz = c["grid"]
    L = 10.0
    if x_cells is not None:
        L = L * x_cells / nx
        nx = x_cells
    return kuhn_beam(nx, ny, nz, L=L, W=1.0, H=1.0, jitter=c.get("jitter", 0.0),
                     jitter_seed=c.get("jitter_seed", 0), node_perm_seed=c.get("node_perm_seed"),
                     tet_perm_seed=c.get("tet_perm_seed"))


def kuhn_counts(nx: int, ny: int, nz: int) -> dict:
    """Closed-form topology counts of the Kuhn beam."""
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    nt = 6 * nx * ny * nz
    ne = 4 * (nx * ny + ny * nz + nz * nx)
    ni = 12 * nx * ny * nz - ne // 2
    edges = (nx * (ny + 1) * (nz + 1) + (nx + 1) * ny * (nz + 1) + (nx + 1) * (ny + 1) * nz
             + nx * ny * (nz + 1) + nx * (ny + 1) * nz + (nx + 1) * ny * nz + nx * ny * nz)
    return dict(n_nodes=nn, n_tets=nt, n_faces=ni + ne, n_interior=ni, n_exterior=ne, n_edges=edges,
                nnz_fs=9 * (nn + 2 * (edges + 6 * nx * ny * nz)), nnz_fem=9 * (nn + 2 * edges),
                eq12_slots=225 * ni + 144 * ne, sum_nf=5 * ni + 4 * ne, sum_nf2=25 * ni + 16 * ne)
