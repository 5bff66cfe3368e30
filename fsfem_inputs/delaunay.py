"""Seeded unstructured tetrahedral beams (stand-in for the paper's TetGen meshes, PAPER.md:545-559,
Table 3): scipy's Delaunay tetrahedralisation of a jittered point lattice, slivers dropped.

Mesh generation only (like TetGen's quality filter) -- no FS-FEM arithmetic: the sliver filter
drops tets whose |signed parallelepiped volume| is below `drop` x the mean, unused points are
removed and ids compacted.  `relabel="degree"` renumbers the nodes by descending node-graph
degree (a deliberately unbanded numbering whose first rows have more than 32 upper-triangle
neighbours -- the generic assembly path).
"""
from __future__ import annotations

import numpy as np

from .kuhn_beam import BeamMesh


def delaunay_beam(nx: int, ny: int, nz: int, L: float = 4.0, W: float = 1.0, H: float = 1.0, jitter: float = 0.3,
                  seed: int = 0, drop: float = 0.02, relabel: str | None = None) -> BeamMesh:
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(seed)
    x, y, z = np.meshgrid(np.linspace(0, L, nx + 1), np.linspace(0, W, ny + 1), np.linspace(0, H, nz + 1),
                          indexing="ij")
    P = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)
    h = np.array([L / nx, W / ny, H / nz])
    inner = (P[:, 0] > 0) & (P[:, 0] < L) & (P[:, 1] > 0) & (P[:, 1] < W) & (P[:, 2] > 0) & (P[:, 2] < H)
    P[inner] += rng.uniform(-jitter, jitter, (int(inner.sum()), 3)) * h
    T = Delaunay(P).simplices.astype(np.int64)
    e1, e2, e3 = P[T[:, 1]] - P[T[:, 0]], P[T[:, 2]] - P[T[:, 0]], P[T[:, 3]] - P[T[:, 0]]
    vol6 = np.abs(np.einsum("ij,ij->i", e1, np.cross(e2, e3)))
    T = T[vol6 > drop * vol6.mean()]
    used = np.unique(T)
    remap = -np.ones(len(P), np.int64)
    remap[used] = np.arange(len(used))
    P, T = P[used], remap[T]
    if relabel == "degree":
        # node-graph degree of the FS pattern is not needed: the tet edge degree orders the same way
        edges = np.concatenate([T[:, [a, b]] for a in range(4) for b in range(a + 1, 4)])
        edges = np.unique(np.sort(edges, 1), axis=0)
        deg = np.bincount(edges.ravel(), minlength=len(P))
        order = np.argsort(-deg, kind="stable")
        newid = np.empty_like(order)
        newid[order] = np.arange(len(order))
        P = P[order]
        T = newid[T]
    xyz = np.ascontiguousarray(P, np.float64)
    tets = np.ascontiguousarray(T, np.int32)
    tol = 1e-9 * L
    dirichlet = np.nonzero(xyz[:, 0] <= tol)[0].astype(np.int32)
    tip = np.nonzero(xyz[:, 0] >= L - tol)[0].astype(np.int32)
    loads = np.zeros((len(xyz), 3))
    loads[tip, 2] = -1.0 / len(tip)
    return BeamMesh(xyz=xyz, tets=tets, dirichlet=dirichlet, loads=loads, tip=tip, grid=(nx, ny, nz), dims=(L, W, H),
                    meta={"kind": "delaunay", "seed": seed, "relabel": relabel})
