"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the FS-FEM method (no volumes, gradients,
smoothing, stiffness, solves).  It only lays out a structured grid, splits each
hex into 6 Kuhn/Freudenthal tets, jitters interior nodes, optionally relabels
nodes / reorders tets, and picks the clamped nodes and the tip load.  Recipe:
DESIGN.md "Input recipe" (SURVEY.md 8(d) Generator G0, readings Q16-Q18).
"""
from .kuhn_beam import (  # noqa: F401
    CONFIGS,
    BeamMesh,
    config_mesh,
    kuhn_beam,
    kuhn_counts,
    splitmix64_stream,
    uniform01,
)
from .delaunay import delaunay_beam  # noqa: F401,E402
