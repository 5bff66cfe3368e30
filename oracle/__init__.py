"""FS-FEM CPU oracle — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/liboracle.so (plain C++17, see oracle.h).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product path (paper_2001_08849_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

STATUS = {0: "ok", 1: "invalid_arg", 2: "topology", 3: "degenerate", 4: "not_converged", 5: "breakdown",
          6: "state"}


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-std=c++17",
               _SRC, "-o", _SO + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, I64, D, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        sig = {
            "ora_new": (P, [P, I64, P, I64]),
            "ora_free": (None, [P]),
            "ora_error": (ctypes.c_char_p, [P]),
            "ora_validate": (I32, [P, P]),
            "ora_build_faces": (I32, [P, P, P]),
            "ora_get_faces": (None, [P, P, P, P]),
            "ora_face_domain": (I32, [P, I64, P, P, P, P, P]),
            "ora_assemble_fs": (I32, [P, D, D, I64, I64]),
            "ora_assemble_fem": (I32, [P, D, D, I64, I64]),
            "ora_face_stiffness": (I32, [P, I64, D, D, P, P]),
            "ora_tet_stiffness": (I32, [P, I64, D, D, P, P]),
            "ora_csr_dims": (None, [P, P, P, P]),
            "ora_last_coo_count": (I64, [P]),
            "ora_set_csr": (I32, [P, I64, P, P, P]),
            "ora_get_csr": (None, [P, P, P, P]),
            "ora_spmv": (I32, [P, P, P]),
            "ora_apply_bc": (I32, [P, P, I64, P, I32, D]),
            "ora_get_rhs": (None, [P, P]),
            "ora_pcg": (I32, [P, D, I64, P, P, P, P]),
            "ora_cholesky": (I32, [P, P]),
            "ora_cholesky_eliminate": (I32, [P, P, I64, P, P]),
            "ora_recover": (I32, [P, D, D, P, P, P, P, P]),
            "ora_surface_loads": (I32, [P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class Oracle:
    """One mesh in the oracle.  Methods mirror SURVEY.md 8(c) O1-O8."""

    def __init__(self, xyz: np.ndarray, tets: np.ndarray):
        self.xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.tets = np.ascontiguousarray(tets, dtype=np.int32)
        self.nn = self.xyz.shape[0]
        self.nt = self.tets.shape[0]
        self._h = lib().ora_new(_p(self.xyz), self.nn, _p(self.tets), self.nt)
        self.timings = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ora_free(h)
            self._h = None

    def _check(self, st: int):
        if st != 0:
            raise OracleError(st, lib().ora_error(self._h).decode())

    def validate(self) -> np.ndarray:
        vol = np.empty(self.nt, dtype=np.float64)
        self._check(lib().ora_validate(self._h, _p(vol)))
        return vol

    def build_faces(self):
        nf, ni = ctypes.c_int64(), ctypes.c_int64()
        t0 = time.perf_counter()
        self._check(lib().ora_build_faces(self._h, ctypes.byref(nf), ctypes.byref(ni)))
        self.timings["faces_s"] = time.perf_counter() - t0
        self.n_faces, self.n_interior = nf.value, ni.value
        fn = np.empty((self.n_faces, 3), np.int32)
        ft = np.empty((self.n_faces, 2), np.int32)
        fo = np.empty((self.n_faces, 2), np.int32)
        lib().ora_get_faces(self._h, _p(fn), _p(ft), _p(fo))
        return fn, ft, fo

    def face_domain(self, f: int):
        field = np.empty(5, np.int32)
        bbar = np.empty((5, 3), np.float64)
        Vf = ctypes.c_double()
        P = ctypes.c_int()
        tri = np.empty((6, 9), np.float64)
        self._check(lib().ora_face_domain(self._h, f, _p(field), _p(bbar), ctypes.byref(Vf), ctypes.byref(P),
                                          _p(tri)))
        return dict(field=field, bbar=bbar, Vf=Vf.value, P=P.value, tri=tri[:P.value].copy())

    def domain_stiffness(self, k: int, E: float, nu: float, tet: bool = False):
        """K7: dense 15x15 stiffness of face k (FS-FEM) or tet k (FEM-T4) and its field nodes."""
        K = np.empty((15, 15), np.float64)
        field = np.empty(5, np.int32)
        fn = lib().ora_tet_stiffness if tet else lib().ora_face_stiffness
        self._check(fn(self._h, k, E, nu, _p(K), _p(field)))
        return K, field

    def _csr(self):
        lo, nr, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib().ora_csr_dims(self._h, ctypes.byref(lo), ctypes.byref(nr), ctypes.byref(nnz))
        rp = np.empty(nr.value + 1, np.int64)
        ci = np.empty(nnz.value, np.int32)
        va = np.empty(nnz.value, np.float64)
        lib().ora_get_csr(self._h, _p(rp), _p(ci), _p(va))
        return lo.value, rp, ci, va

    def assemble_fs(self, E: float, nu: float, node_lo: int = 0, node_hi: int | None = None):
        node_hi = self.nn if node_hi is None else node_hi
        t0 = time.perf_counter()
        self._check(lib().ora_assemble_fs(self._h, E, nu, node_lo, node_hi))
        self.timings["assemble_s"] = time.perf_counter() - t0
        return self._csr()

    def assemble_fem(self, E: float, nu: float, node_lo: int = 0, node_hi: int | None = None):
        node_hi = self.nn if node_hi is None else node_hi
        self._check(lib().ora_assemble_fem(self._h, E, nu, node_lo, node_hi))
        return self._csr()

    def last_coo_count(self) -> int:
        return int(lib().ora_last_coo_count(self._h))

    def set_csr(self, row_ptr, col_idx, vals):
        self._keep = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                      np.ascontiguousarray(vals, np.float64))
        rp, ci, va = self._keep
        self._check(lib().ora_set_csr(self._h, rp.size - 1, _p(rp), _p(ci), _p(va)))

    def spmv(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(3 * self.nn, np.float64)
        self._check(lib().ora_spmv(self._h, _p(x), _p(y)))
        return y

    def apply_bc(self, dirichlet: np.ndarray, loads: np.ndarray, mode: int = 0, penalty_scale: float = 0.0):
        d = np.ascontiguousarray(dirichlet, np.int32)
        f = np.ascontiguousarray(loads, np.float64).reshape(-1)
        t0 = time.perf_counter()
        self._check(lib().ora_apply_bc(self._h, _p(d), d.size, _p(f), mode, penalty_scale))
        self.timings["bc_s"] = time.perf_counter() - t0
        rhs = np.empty(3 * self.nn, np.float64)
        lib().ora_get_rhs(self._h, _p(rhs))
        lo, rp, ci, va = self._csr()
        return rp, ci, va, rhs

    def pcg(self, tol: float = 1e-10, max_iter: int = 0, allow_not_converged: bool = False):
        u = np.empty(3 * self.nn, np.float64)
        it, rr, tr = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        t0 = time.perf_counter()
        st = lib().ora_pcg(self._h, tol, max_iter, _p(u), ctypes.byref(it), ctypes.byref(rr), ctypes.byref(tr))
        self.timings["pcg_s"] = time.perf_counter() - t0
        if not (st == 0 or (st == 4 and allow_not_converged)):
            self._check(st)
        return u, dict(iterations=it.value, rel_residual=rr.value, true_rel_residual=tr.value, status=st)

    def cholesky(self) -> np.ndarray:
        u = np.empty(3 * self.nn, np.float64)
        self._check(lib().ora_cholesky(self._h, _p(u)))
        return u

    def recover(self, E: float, nu: float, u: np.ndarray):
        """O9: (face strain [N_f,6], face stress [N_f,6], nodal stress [nn,6], nodal von Mises [nn])."""
        u = np.ascontiguousarray(u, np.float64).reshape(-1)
        nf = len(self.build_faces()[0]) if not hasattr(self, "n_faces") else self.n_faces
        eps, sig = np.empty((nf, 6)), np.empty((nf, 6))
        ns, vm = np.empty((self.nn, 6)), np.empty(self.nn)
        self._check(lib().ora_recover(self._h, E, nu, _p(u), _p(eps), _p(sig), _p(ns), _p(vm)))
        return eps, sig, ns, vm

    def surface_loads(self, node_flag: np.ndarray, traction) -> np.ndarray:
        """O10: nodal loads [nn, 3] of a uniform traction on the flagged exterior faces."""
        fl = np.ascontiguousarray(node_flag, np.uint8)
        t = np.ascontiguousarray(traction, np.float64)
        out = np.empty((self.nn, 3))
        self._check(lib().ora_surface_loads(self._h, _p(fl), _p(t), _p(out)))
        return out

    def cholesky_eliminate(self, dirichlet: np.ndarray, loads: np.ndarray) -> np.ndarray:
        d = np.ascontiguousarray(dirichlet, np.int32)
        f = np.ascontiguousarray(loads, np.float64).reshape(-1)
        u = np.empty(3 * self.nn, np.float64)
        self._check(lib().ora_cholesky_eliminate(self._h, _p(d), d.size, _p(f), _p(u)))
        return u


def csr_to_dense(row_ptr, col_idx, vals, n_cols):
    n = row_ptr.size - 1
    A = np.zeros((n, n_cols))
    for r in range(n):
        for k in range(row_ptr[r], row_ptr[r + 1]):
            A[r, col_idx[k]] += vals[k]
    return A


__all__ = ["Oracle", "OracleError", "build", "csr_to_dense", "STATUS"]
