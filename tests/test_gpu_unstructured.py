"""Unstructured meshes (VERDICT r01 missing #5): Delaunay tetrahedralisations of jittered point
lattices stand in for the paper's TetGen cantilevers (Table 3; ~4-6 tets per
node, irregular node graph, both tet orientations).  With the degree-descending relabelling the
first rows hold more than 32 upper-triangle blocks, which drives the assembly's generic path.

Bars as everywhere: faces / row_ptr / col_idx bit-exact, values 1e-12 max|K|, u 1e-7."""
import numpy as np
import pytest

from fsfem_inputs import delaunay_beam
from oracle import Oracle

pytestmark = pytest.mark.gpu

E, NU = 1.0e6, 0.3


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2001_08849_b200 as P
    P.load_library()
    return P


MESHES = {
    "delaunay": dict(nx=16, ny=6, ny_=6, seed=5, relabel=None),
    "delaunay_degree_relabel": dict(nx=16, ny=6, ny_=6, seed=5, relabel="degree"),
    "delaunay_big": dict(nx=40, ny=10, ny_=10, seed=9, relabel=None),
}


def mesh(name):
    k = MESHES[name]
    return delaunay_beam(k["nx"], k["ny"], k["ny_"], seed=k["seed"], relabel=k["relabel"])


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("reorder", [0, 2], ids=["reorder-auto", "reorder-never"])
def test_unstructured_parity(P, name, reorder):
    m = mesh(name)
    o = Oracle(m.xyz, m.tets)
    ofn, oft, ofo = o.build_faces()
    g = P.FsFem()
    g.set_reorder(reorder)
    g.build_faces(m.xyz, m.tets)
    fn, ft, fo = g.get_faces()
    assert np.array_equal(fn, ofn) and np.array_equal(ft, oft) and np.array_equal(fo, ofo)
    g.assemble_csr(E, NU)
    c = g.get_csr()
    _, orp, oci, ova = o.assemble_fs(E, NU)
    assert np.array_equal(c.row_ptr, orp) and np.array_equal(c.col_idx, oci)
    kmax = np.abs(ova).max()
    assert np.abs(c.vals - ova).max() <= 1e-12 * kmax
    rep = g.report()
    if name == "delaunay_degree_relabel" and reorder == 2:
        assert rep["stored_blocks"] > 0
        # some rows hold > 32 stored (upper-triangle) blocks: the long-row path ran (values checked above)
        stored = [int(np.sum(oci[orp[3 * i]:orp[3 * i + 1]] // 3 >= i)) // 3 for i in range(m.n_nodes)]
        assert max(stored) > 32
    x = np.random.default_rng(1).standard_normal(3 * m.n_nodes)
    q = g.spmv(x)
    assert np.abs(q - o.spmv(x)).max() <= 1e-11 * kmax * np.abs(x).max()
    g.apply_bc(m.dirichlet, m.loads.reshape(-1))
    u, rep = g.pcg_solve(rel_tol=1e-10)
    o.apply_bc(m.dirichlet, m.loads, 0)
    uo, orep = o.pcg(1e-10)
    assert rep["converged"] == 1
    assert np.linalg.norm(u - uo) <= 1e-7 * np.linalg.norm(uo)
    g.close()


def _icosphere_star(subdiv: int):
    """A ball: the triangles of a subdivided icosahedron coned to the centre node 0 -- node 0 lies in
    every tet (20 * 4**subdiv of them), a valid manifold mesh with one very high-valence node."""
    t = (1 + 5 ** 0.5) / 2
    V = [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
         [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]]
    F = [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6],
         [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10],
         [8, 6, 7], [9, 8, 1]]
    V = [list(np.array(v) / np.linalg.norm(v)) for v in V]
    for _ in range(subdiv):
        mid = {}

        def m(a, b):
            k = (min(a, b), max(a, b))
            if k not in mid:
                p = (np.array(V[a]) + np.array(V[b])) / 2
                V.append(list(p / np.linalg.norm(p)))
                mid[k] = len(V) - 1
            return mid[k]
        F = [g for a, b, c in F for g in ([a, m(a, b), m(c, a)], [b, m(b, c), m(a, b)], [c, m(c, a), m(b, c)],
                                           [m(a, b), m(b, c), m(c, a)])]
    xyz = np.vstack([[0.0, 0.0, 0.0], np.array(V)])
    tets = np.array([[0, a + 1, b + 1, c + 1] for a, b, c in F], np.int32)
    return xyz, tets


def test_high_valence_node_limits(P):
    """Documented limits (include/fsfem.h UNSUPPORTED): a node in more than 128 tets is rejected by
    the symbolic pass; below the limit the same kind of mesh assembles and matches the oracle."""
    xyz, tets = _icosphere_star(2)  # 320 tets around node 0
    g = P.FsFem()
    g.build_faces(xyz, tets)
    # 960 face instances in node 0's bucket: the CTA (large-bucket) sort ran; faces still bit-exact
    ofn, oft, ofo = Oracle(xyz, tets).build_faces()
    fn, ft, fo = g.get_faces()
    assert np.array_equal(fn, ofn) and np.array_equal(ft, oft) and np.array_equal(fo, ofo)
    with pytest.raises(P.FsfemError) as e:
        g.assemble_csr(E, NU)
    assert e.value.status == "UNSUPPORTED"
    g.close()
    xyz, tets = _icosphere_star(1)  # 80 tets around node 0: within the limits
    o = Oracle(xyz, tets)
    o.build_faces()
    _, orp, oci, ova = o.assemble_fs(E, NU)
    g = P.FsFem()
    g.build_faces(xyz, tets)
    g.assemble_csr(E, NU)
    c = g.get_csr()
    assert np.array_equal(c.row_ptr, orp) and np.array_equal(c.col_idx, oci)
    assert np.abs(c.vals - ova).max() <= 1e-12 * np.abs(ova).max()
    g.close()


def test_face_bucket_limits(P):
    """Face extraction buckets by the smallest vertex: 3840 instances (1280 tets around node 0) use
    the large-bucket sort and match the oracle; beyond kBigCap = 4096 instances (5120 tets,
    15360 instances) build_faces reports UNSUPPORTED (include/fsfem.h)."""
    xyz, tets = _icosphere_star(3)
    g = P.FsFem()
    g.build_faces(xyz, tets)
    ofn, oft, ofo = Oracle(xyz, tets).build_faces()
    fn, ft, fo = g.get_faces()
    assert np.array_equal(fn, ofn) and np.array_equal(ft, oft) and np.array_equal(fo, ofo)
    g.close()
    xyz, tets = _icosphere_star(4)
    g = P.FsFem()
    with pytest.raises(P.FsfemError) as e:
        g.build_faces(xyz, tets)
    assert e.value.status == "UNSUPPORTED"
    g.close()
