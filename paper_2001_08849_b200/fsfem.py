"""Thin ctypes binding of libfsfem.so (include/fsfem.h): argument marshalling only.

Every step of the path runs in the library's sm_100a kernels.  There is no CPU fallback:
if the shared library is missing or cannot be loaded, importing/calling raises.
Arrays may be numpy arrays (host) or torch tensors (host or CUDA); the library detects
host vs device pointers itself (include/fsfem.h, "Memory").
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfsfem.so")
# Tuning experiments may point at another build of the same sources (scripts/, never the tests).
if os.environ.get("FSFEM_LIB"):
    LIB_PATH = os.path.abspath(os.environ["FSFEM_LIB"])

STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "TOPOLOGY", 3: "DEGENERATE", 4: "UNSUPPORTED", 5: "NOT_CONVERGED",
                6: "BREAKDOWN", 7: "STATE", 8: "CUDA", 9: "NCCL", 10: "OOM"}

# Every symbol include/fsfem.h declares (checked by tests/test_abi.py).
METHOD_FS, METHOD_FEM_T4 = 0, 1

EXPORTS = ["fsfem_status_string", "fsfem_create", "fsfem_destroy", "fsfem_last_error", "fsfem_comm_init",
           "fsfem_comm_init_loopback", "fsfem_get_partition", "fsfem_set_deterministic", "fsfem_set_loop", "fsfem_set_overlap", "fsfem_set_method", "fsfem_set_reorder", "fsfem_set_pcg_variant", "fsfem_set_exchange", "fsfem_get_halo",
           "fsfem_nccl_get_unique_id", "fsfem_build_faces", "fsfem_get_faces", "fsfem_assemble_csr",
           "fsfem_get_csr", "fsfem_apply_bc", "fsfem_pcg_solve", "fsfem_get_report", "fsfem_spmv", "fsfem_recover_stress",
           "fsfem_surface_loads", "fsfem_domain_stiffness"]


class FsfemReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("converged", ctypes.c_int32), ("reordered", ctypes.c_int32),
                ("rel_residual", ctypes.c_double), ("true_rel_residual", ctypes.c_double),
                ("t_faces_ms", ctypes.c_double), ("t_symbolic_ms", ctypes.c_double),
                ("t_numeric_ms", ctypes.c_double), ("t_bc_ms", ctypes.c_double), ("t_pcg_ms", ctypes.c_double),
                ("t_spmv_ms", ctypes.c_double), ("spmv_launches", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("stored_blocks", ctypes.c_int64),
                ("transposed_blocks", ctypes.c_int64), ("spmv_bytes", ctypes.c_int64),
                ("assembly_bytes", ctypes.c_int64), ("spmv_kernel", ctypes.c_int64),
                ("residual_floor", ctypes.c_double), ("restarts", ctypes.c_int64),
                ("assembly_aux_bytes", ctypes.c_int64), ("t_spmv_dev_ms", ctypes.c_double),
                ("spmv_dev_launches", ctypes.c_int64), ("pcg_loop", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class FsfemError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fsfem {STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS_NAMES.get(code, str(code))


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libfsfem.so (raises OSError if it is missing: build it with paper_2001_08849_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not found: run `python -m paper_2001_08849_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    sig = {
        "fsfem_status_string": (ctypes.c_char_p, [I]),
        "fsfem_create": (I, [I, P, ctypes.POINTER(P)]),
        "fsfem_destroy": (I, [P]),
        "fsfem_last_error": (ctypes.c_char_p, [P]),
        "fsfem_comm_init": (I, [P, P, I, I]),
        "fsfem_comm_init_loopback": (I, [P, I]),
        "fsfem_get_partition": (I, [P, P]),
        "fsfem_set_deterministic": (I, [P, I]),
        "fsfem_set_loop": (I, [P, I]),
        "fsfem_set_overlap": (I, [P, I]),
        "fsfem_set_method": (I, [P, I]),
        "fsfem_set_reorder": (I, [P, I]),
        "fsfem_set_pcg_variant": (I, [P, I]),
        "fsfem_set_exchange": (I, [P, I]),
        "fsfem_get_halo": (I, [P, P, P]),
        "fsfem_nccl_get_unique_id": (I, [P]),
        "fsfem_build_faces": (I, [P, P, I64, P, I64, P, P]),
        "fsfem_get_faces": (I, [P, P, P, P]),
        "fsfem_assemble_csr": (I, [P, D, D, P, P, P]),
        "fsfem_get_csr": (I, [P, P, P, P]),
        "fsfem_apply_bc": (I, [P, P, I64, P, I, D]),
        "fsfem_pcg_solve": (I, [P, P, I, D, I64, ctypes.POINTER(FsfemReport)]),
        "fsfem_get_report": (I, [P, ctypes.POINTER(FsfemReport)]),
        "fsfem_spmv": (I, [P, P, P]),
        "fsfem_recover_stress": (I, [P, P, P, P, P, P, P]),
        "fsfem_domain_stiffness": (I, [P, P, ctypes.c_int64, P, P]),
        "fsfem_surface_loads": (I, [P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (host or device); None -> NULL."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    raise TypeError(f"unsupported array type {type(a)}")


def _check_dtype(a, np_dtype, name):
    if a is None:
        return
    if isinstance(a, np.ndarray):
        if a.dtype != np_dtype:
            raise TypeError(f"{name} must be {np.dtype(np_dtype).name}, got {a.dtype}")
    else:
        want = {np.float64: "torch.float64", np.int32: "torch.int32", np.int64: "torch.int64"}[np_dtype]
        if str(a.dtype) != want:
            raise TypeError(f"{name} must be {want}, got {a.dtype}")


def _nelem(a):
    return a.size if isinstance(a, np.ndarray) else a.numel()


# ------------------------------------------------------------------ C-ABI mirror (same names)
def fsfem_create(cuda_device: int = 0, cuda_stream: int | None = None):
    L = load_library()
    h = ctypes.c_void_p()
    st = L.fsfem_create(cuda_device, ctypes.c_void_p(cuda_stream) if cuda_stream else None, ctypes.byref(h))
    if st != 0:
        raise FsfemError(st, "fsfem_create failed")
    return h


def fsfem_destroy(ctx) -> None:
    load_library().fsfem_destroy(ctx)


def _raise(ctx, st):
    if st != 0:
        raise FsfemError(st, load_library().fsfem_last_error(ctx).decode())


def fsfem_nccl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = load_library().fsfem_nccl_get_unique_id(buf)
    if st != 0:
        raise FsfemError(st, "ncclGetUniqueId failed")
    return buf.raw


def fsfem_comm_init(ctx, unique_id: bytes | None, rank: int, nranks: int) -> None:
    """unique_id None: partition-only context (include/fsfem.h)."""
    buf = ctypes.create_string_buffer(bytes(unique_id), 128) if unique_id is not None else None
    _raise(ctx, load_library().fsfem_comm_init(ctx, buf, rank, nranks))


def fsfem_comm_init_loopback(ctxs) -> None:
    """Make the contexts ctxs[0..n) ranks 0..n-1 of one in-process loopback group (include/fsfem.h)."""
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value if isinstance(c, ctypes.c_void_p) else c for c in ctxs])
    st = load_library().fsfem_comm_init_loopback(arr, len(ctxs))
    if st != 0:
        _raise(ctxs[0], st)


def fsfem_get_partition(ctx, nranks: int) -> np.ndarray:
    out = np.zeros(nranks + 1, np.int64)
    _raise(ctx, load_library().fsfem_get_partition(ctx, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def fsfem_set_loop(ctx, mode: int) -> None:
    """0: device-side while loop, 1: host-polled graph batches, 2: one thread-block-cluster launch,
    3: auto (default: cluster for small meshes, else host batches)."""
    _raise(ctx, load_library().fsfem_set_loop(ctx, int(mode)))


def fsfem_set_overlap(ctx, on: bool) -> None:
    """Exchange of the search direction overlapped with the interior rows' SpMV (multi-rank)."""
    _raise(ctx, load_library().fsfem_set_overlap(ctx, 1 if on else 0))


def fsfem_set_deterministic(ctx, on: bool) -> None:
    _raise(ctx, load_library().fsfem_set_deterministic(ctx, 1 if on else 0))


def fsfem_set_method(ctx, method: int) -> None:
    _raise(ctx, load_library().fsfem_set_method(ctx, int(method)))


def fsfem_set_pcg_variant(ctx, variant: int) -> None:
    """0: standard PCG recurrence, 1: single reduction per iteration (Chronopoulos-Gear),
    2: auto (default: the standard recurrence)."""
    _raise(ctx, load_library().fsfem_set_pcg_variant(ctx, int(variant)))


def fsfem_set_exchange(ctx, mode: int) -> None:
    """0: all-gather of the search direction (default), 1: halo-only send/recv."""
    _raise(ctx, load_library().fsfem_set_exchange(ctx, int(mode)))


def fsfem_get_halo(ctx) -> np.ndarray:
    """The rank's halo node ids (ascending); empty with one rank."""
    lib = load_library()
    n = ctypes.c_int64(0)
    _raise(ctx, lib.fsfem_get_halo(ctx, None, ctypes.byref(n)))
    out = np.zeros(max(n.value, 0), np.int32)
    if n.value > 0:
        _raise(ctx, lib.fsfem_get_halo(ctx, out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)))
    return out


def fsfem_set_reorder(ctx, mode: int) -> None:
    """0 auto (default), 1 always, 2 never (include/fsfem.h)."""
    _raise(ctx, load_library().fsfem_set_reorder(ctx, int(mode)))


def fsfem_build_faces(ctx, xyz, tets):
    _check_dtype(xyz, np.float64, "xyz")
    _check_dtype(tets, np.int32, "tets")
    nf, ni = ctypes.c_int64(), ctypes.c_int64()
    _raise(ctx, load_library().fsfem_build_faces(ctx, _ptr(xyz), _nelem(xyz) // 3, _ptr(tets), _nelem(tets) // 4,
                                                 ctypes.byref(nf), ctypes.byref(ni)))
    return nf.value, ni.value


def fsfem_get_faces(ctx, face_nodes, face_tet, face_opp) -> None:
    _raise(ctx, load_library().fsfem_get_faces(ctx, _ptr(face_nodes), _ptr(face_tet), _ptr(face_opp)))


def fsfem_assemble_csr(ctx, E: float, nu: float):
    rb, nr, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _raise(ctx, load_library().fsfem_assemble_csr(ctx, E, nu, ctypes.byref(rb), ctypes.byref(nr), ctypes.byref(nnz)))
    return rb.value, nr.value, nnz.value


def fsfem_get_csr(ctx, row_ptr, col_idx, vals) -> None:
    _raise(ctx, load_library().fsfem_get_csr(ctx, _ptr(row_ptr), _ptr(col_idx), _ptr(vals)))


def fsfem_apply_bc(ctx, dirichlet_nodes, loads, mode: int = 0, penalty_scale: float = 0.0) -> None:
    _check_dtype(dirichlet_nodes, np.int32, "dirichlet_nodes")
    _check_dtype(loads, np.float64, "loads")
    _raise(ctx, load_library().fsfem_apply_bc(ctx, _ptr(dirichlet_nodes), _nelem(dirichlet_nodes), _ptr(loads), mode,
                                              penalty_scale))


def fsfem_pcg_solve(ctx, u, u0_is_zero: bool = True, rel_tol: float = 1e-10, max_iter: int = 0,
                    allow_not_converged: bool = False) -> dict:
    _check_dtype(u, np.float64, "u")
    rep = FsfemReport()
    st = load_library().fsfem_pcg_solve(ctx, _ptr(u), 1 if u0_is_zero else 0, rel_tol, max_iter, ctypes.byref(rep))
    d = rep.as_dict()
    d["status"] = STATUS_NAMES.get(st, st)
    if st != 0 and not (st == 5 and allow_not_converged):
        _raise(ctx, st)
    return d


def fsfem_get_report(ctx) -> dict:
    rep = FsfemReport()
    _raise(ctx, load_library().fsfem_get_report(ctx, ctypes.byref(rep)))
    return rep.as_dict()


def fsfem_spmv(ctx, p, q) -> None:
    _raise(ctx, load_library().fsfem_spmv(ctx, _ptr(p), _ptr(q)))


def fsfem_recover_stress(ctx, u, strain, stress, node_stress, node_vm) -> int:
    nd = ctypes.c_int64()
    _raise(ctx, load_library().fsfem_recover_stress(ctx, _ptr(u), _ptr(strain), _ptr(stress), _ptr(node_stress),
                                                    _ptr(node_vm), ctypes.byref(nd)))
    return nd.value


def fsfem_domain_stiffness(ctx, ids, K, field) -> None:
    _raise(ctx, load_library().fsfem_domain_stiffness(ctx, _ptr(ids), _nelem(ids), _ptr(K), _ptr(field)))


def fsfem_surface_loads(ctx, node_flag, traction, loads) -> None:
    t = np.ascontiguousarray(traction, np.float64)
    _raise(ctx, load_library().fsfem_surface_loads(ctx, _ptr(node_flag), _ptr(t), _ptr(loads)))


# ------------------------------------------------------------------ convenience object
@dataclass
class Csr:
    row_begin: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray


class FsFem:
    """One context = one mesh on one GPU (one rank).  Host numpy in, host numpy out."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.ctx = fsfem_create(device, stream)
        self.n_nodes = self.n_faces = self.n_interior = 0

    def close(self):
        if getattr(self, "ctx", None):
            fsfem_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def comm_init(self, unique_id: bytes | None, rank: int, nranks: int):
        fsfem_comm_init(self.ctx, unique_id, rank, nranks)
        self.nranks = nranks

    def partition(self) -> np.ndarray:
        return fsfem_get_partition(self.ctx, getattr(self, "nranks", 1))

    def set_deterministic(self, on: bool = True):
        fsfem_set_deterministic(self.ctx, on)

    def set_loop(self, mode: int):
        fsfem_set_loop(self.ctx, mode)

    def set_overlap(self, on: bool = True):
        fsfem_set_overlap(self.ctx, on)

    def set_reorder(self, mode: int):
        fsfem_set_reorder(self.ctx, mode)

    def set_pcg_variant(self, variant: int):
        fsfem_set_pcg_variant(self.ctx, variant)

    def set_exchange(self, mode: int):
        fsfem_set_exchange(self.ctx, mode)

    def halo(self) -> np.ndarray:
        return fsfem_get_halo(self.ctx)

    def set_method(self, method: int):
        fsfem_set_method(self.ctx, method)

    def build_faces(self, xyz, tets):
        self.n_nodes = _nelem(xyz) // 3
        self.n_faces, self.n_interior = fsfem_build_faces(self.ctx, xyz, tets)
        return self.n_faces, self.n_interior

    def get_faces(self):
        fn = np.empty((self.n_faces, 3), np.int32)
        ft = np.empty((self.n_faces, 2), np.int32)
        fo = np.empty((self.n_faces, 2), np.int32)
        fsfem_get_faces(self.ctx, fn, ft, fo)
        return fn, ft, fo

    def assemble_csr(self, E: float, nu: float):
        self.row_begin, self.n_rows, self.nnz = fsfem_assemble_csr(self.ctx, E, nu)
        return self.row_begin, self.n_rows, self.nnz

    def get_csr(self, with_pattern: bool = True) -> Csr:
        rp = np.empty(self.n_rows + 1, np.int64) if with_pattern else None
        ci = np.empty(self.nnz, np.int32) if with_pattern else None
        va = np.empty(self.nnz, np.float64)
        fsfem_get_csr(self.ctx, rp, ci, va)
        return Csr(self.row_begin, rp, ci, va)

    def apply_bc(self, dirichlet_nodes, loads, mode: int = 0, penalty_scale: float = 0.0):
        fsfem_apply_bc(self.ctx, dirichlet_nodes, loads, mode, penalty_scale)

    def pcg_solve(self, u0=None, rel_tol: float = 1e-10, max_iter: int = 0, allow_not_converged: bool = False):
        u = np.zeros(3 * self.n_nodes) if u0 is None else np.ascontiguousarray(u0, np.float64).reshape(-1).copy()
        rep = fsfem_pcg_solve(self.ctx, u, u0 is None, rel_tol, max_iter, allow_not_converged)
        return u, rep

    def spmv(self, p):
        q = np.zeros(3 * self.n_nodes)
        fsfem_spmv(self.ctx, np.ascontiguousarray(p, np.float64), q)
        return q

    def recover_stress(self, u, n_domains: int):
        """(domain strain [n,6], domain stress [n,6], nodal stress [nn,6], nodal von Mises [nn])."""
        u = np.ascontiguousarray(u, np.float64).reshape(-1)
        eps, sig = np.empty((n_domains, 6)), np.empty((n_domains, 6))
        ns, vm = np.zeros((self.n_nodes, 6)), np.zeros(self.n_nodes)
        fsfem_recover_stress(self.ctx, u, eps, sig, ns, vm)
        return eps, sig, ns, vm

    def domain_stiffness(self, ids):
        """K7 debug export: (K [n, 15, 15], field [n, 5]) of faces (FS-FEM) or tets (FEM-T4) ids."""
        ids = np.ascontiguousarray(ids, np.int64).reshape(-1)
        K = np.empty((len(ids), 15, 15))
        field = np.empty((len(ids), 5), np.int32)
        fsfem_domain_stiffness(self.ctx, ids, K, field)
        return K, field

    def surface_loads(self, node_flag, traction):
        """Nodal loads [n_nodes, 3] of a uniform traction on the flagged exterior faces."""
        loads = np.zeros((self.n_nodes, 3))
        fsfem_surface_loads(self.ctx, np.ascontiguousarray(node_flag, np.uint8), traction, loads)
        return loads

    def report(self) -> dict:
        return fsfem_get_report(self.ctx)
