"""B200 (sm_100a) FS-FEM hot path: faces -> smoothed stiffness (CSR) -> BCs -> Jacobi-PCG.

The compute lives in libfsfem.so (csrc/*.cu, C ABI in include/fsfem.h); fsfem.py is a ctypes
binding.  Method: arxiv 2001.08849 (juSFEM), see DESIGN.md.
"""
from .fsfem import (  # noqa: F401
    EXPORTS,
    METHOD_FEM_T4,
    METHOD_FS,
    LIB_PATH,
    Csr,
    FsFem,
    FsfemError,
    fsfem_apply_bc,
    fsfem_assemble_csr,
    fsfem_build_faces,
    fsfem_comm_init,
    fsfem_comm_init_loopback,
    fsfem_get_partition,
    fsfem_set_deterministic,
    fsfem_set_loop,
    fsfem_set_overlap,
    fsfem_create,
    fsfem_destroy,
    fsfem_get_csr,
    fsfem_get_faces,
    fsfem_get_report,
    fsfem_nccl_get_unique_id,
    fsfem_pcg_solve,
    fsfem_recover_stress,
    fsfem_set_method,
    fsfem_set_reorder,
    fsfem_set_pcg_variant,
    fsfem_set_exchange,
    fsfem_get_halo,
    fsfem_spmv,
    fsfem_surface_loads,
    load_library,
)
