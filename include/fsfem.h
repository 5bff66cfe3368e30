/* fsfem.h — C ABI of the B200 (sm_100a) FS-FEM hot path.
 *
 * Method: face-based smoothed FEM (FS-FEM) for 3D linear elasticity on 4-node tetrahedra,
 * arxiv 2001.08849 (juSFEM), §2.1 STEPs 1-5 (lines 124-245) and §3.2-3.3 (303-449).
 * The library computes, on one GPU per process:
 *   S1  the unique faces (smoothing domains) of the mesh         (Alg. 1)
 *   S2-S4 per-face smoothed gradients b_I and V_f                  (Eqs. 2-7)
 *   S5-S6 the global smoothed stiffness K = sum_f B^T c B V_f     (Eqs. 8-9)
 *         as CSR with a fixed (deterministic) summation order
 *   S7  essential boundary conditions
 *   S8-S9 K d = f by Jacobi-preconditioned CG                     (replaces PARDISO)
 *
 * Conventions:
 *   - dof numbering: dof = 3*node + component (x, y, z)                                (Q12)
 *   - material: isotropic, Voigt (xx, yy, zz, yz, xz, xy), engineering shear strains   (Q1)
 *   - faces are ordered by their sorted vertex triple (a < b < c); an interior face lists
 *     its two tets with t0 < t1; exterior faces have t1 = opp1 = -1                     (Q11)
 *   - CSR keeps every structural entry (full 3x3 blocks for every pair of nodes sharing a
 *     smoothing domain), columns ascending                                             (Q13)
 *   - either tet orientation is accepted (volumes use |det|)                           (Q6)
 *
 * Memory: every array argument may point to HOST memory (pageable or pinned) or to DEVICE
 * memory of the context's device; the library tells them apart with cudaPointerGetAttributes
 * and copies host data in/out itself (copies are stream-ordered on the context stream).
 * The caller owns all its buffers; the context owns every intermediate it allocates until
 * fsfem_destroy or the next fsfem_build_faces.  Calls are asynchronous on the context stream
 * except where they return host scalars, which synchronize that stream.  No C++ exception
 * crosses the ABI; every call returns an fsfem_status and fsfem_last_error() explains it.
 *
 * Call order: create -> [comm_init] -> build_faces -> assemble_csr -> apply_bc -> pcg_solve.
 * A violation returns FSFEM_ERR_STATE.  Re-calling assemble_csr re-runs only the numeric
 * assembly (S6) on the cached pattern; it invalidates earlier BCs.
 */
#ifndef FSFEM_H
#define FSFEM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FSFEM_OK = 0,
  FSFEM_ERR_INVALID_ARG = 1,   /* null pointer, size <= 0, node id out of range, E <= 0,
                                  nu outside (-1, 0.5), bad mode, unknown pointer kind       */
  FSFEM_ERR_TOPOLOGY = 2,      /* a face shared by more than two tets (non-manifold mesh)    */
  FSFEM_ERR_DEGENERATE = 3,    /* a tet repeats a node or |V_e| <= 1e-14 * diag(bbox)^3      */
  FSFEM_ERR_UNSUPPORTED = 4,   /* n_nodes >= 2^31/3, nnz >= 2^31, a node in > 4096 faces, ... */
  FSFEM_ERR_NOT_CONVERGED = 5, /* max_iter reached: u holds the last iterate, report filled   */
  FSFEM_ERR_BREAKDOWN = 6,     /* non-finite value or p.q <= 0 in PCG (K not SPD after BCs)  */
  FSFEM_ERR_STATE = 7,         /* call order violated                                        */
  FSFEM_ERR_CUDA = 8,          /* a CUDA runtime error (message has the CUDA error string)   */
  FSFEM_ERR_NCCL = 9,          /* an NCCL error                                              */
  FSFEM_ERR_OOM = 10           /* device allocation failed                                   */
} fsfem_status;

typedef struct fsfem_ctx fsfem_ctx; /* opaque */

typedef struct {
  int64_t iterations;        /* PCG iterations performed (SpMVs inside the loop)            */
  int32_t converged;         /* 1 if ||r||_2 <= rel_tol * ||f||_2 was reached               */
  int32_t reordered;         /* 1 if the last build_faces renumbered the nodes internally     */
  double rel_residual;       /* recurrence residual ||r|| / ||f|| at exit                    */
  double true_rel_residual;  /* ||f - K u|| / ||f|| recomputed at exit                       */
  double t_faces_ms;         /* device time (CUDA events) of the last build_faces (S1)       */
  double t_symbolic_ms;      /* ... of the symbolic CSR pass (S5, first assemble only)       */
  double t_numeric_ms;       /* ... of the last numeric assembly (S2-S4, S6)                 */
  double t_bc_ms;            /* ... of the last apply_bc (S7)                                */
  double t_pcg_ms;           /* ... of the last pcg_solve loop (S8-S9)                       */
  double t_spmv_ms;          /* summed CUDA-event time of the sampled PCG SpMV launches (the first
                                SpMV of every graph batch; device loop: = t_spmv_dev_ms)        */
  int64_t spmv_launches;     /* number of SpMV launches in t_spmv_ms                          */
  int64_t kernel_launches;   /* kernels launched by libfsfem in this process so far (monotonic;
                                graph replays count their kernels, early-exit ones included) */
  /* Storage and algorithmic traffic of the assembled operator.  K is stored as
   * its symmetric half: stored_blocks 3x3 blocks (j >= i, plus halo columns of other ranks) and
   * transposed_blocks located through a list.                                                 */
  int64_t stored_blocks;
  int64_t transposed_blocks;
  int64_t spmv_bytes;        /* minimum DRAM bytes of one SpMV launch: stored values, column ids,
                                transposed list, row pointers, x read once, y written once       */
  int64_t assembly_bytes;    /* minimum DRAM bytes of one numeric assembly: mesh read + stored
                                values written                                                   */
  int64_t spmv_kernel;       /* SpMV kernel of this pattern: 0 warp per node (small meshes),
                                1 gather (transposed blocks read from their rows), 2 dataflow push
                                                                                   */
  double residual_floor;     /* rounding floor of the true residual at exit:
                                2^-52 * ||K||_F * ||u||_2 / ||f||_2 (||K||_F bounded from above)   */
  int64_t restarts;          /* residual-replacement restarts of the last pcg_solve              */
  int64_t assembly_aux_bytes; /* bytes of the precomputed assembly tiles read per numeric assembly
                                 (domain lists, field positions, block programs)   */
  double t_spmv_dev_ms;      /* summed duration of EVERY PCG SpMV launch of the solve, timed on the
                                device (%globaltimer: first CTA start to last CTA end)          */
  int64_t spmv_dev_launches; /* number of launches in t_spmv_dev_ms                              */
  int64_t pcg_loop;          /* loop that ran the last pcg_solve: FSFEM_LOOP_DEVICE, _HOST or
                                _CLUSTER (see fsfem_set_loop)                                     */
} fsfem_report;

/* Human-readable name of a status code (static string). */
const char* fsfem_status_string(fsfem_status s);

/* Create a context on CUDA device `cuda_device`.  `cuda_stream` is a cudaStream_t (e.g.
 * torch.cuda.current_stream().cuda_stream) or NULL, in which case the context creates its own
 * non-blocking stream.  *out receives the context. */
fsfem_status fsfem_create(int cuda_device, void* cuda_stream, fsfem_ctx** out);
/* Frees every device buffer of the context.  NULL-safe. */
fsfem_status fsfem_destroy(fsfem_ctx* ctx);
/* Last error message of the context ("" if none); valid until the next call on ctx. */
const char* fsfem_last_error(const fsfem_ctx* ctx);

/* Multi-GPU: join an NCCL communicator of `nranks` processes, one GPU each.
 * `nccl_unique_id` is the 128-byte ncclUniqueId (host memory) created by rank 0 and
 * broadcast by the caller.  Rank r then owns the contiguous node range
 * [ranges[r], ranges[r+1]) (fsfem_get_partition) and builds only those rows.  The ranges are
 * computed at build_faces, identically on every rank, so that the node-face incidences (the
 * rows' share of assembly work and nnz) are balanced; they are aligned to 32 nodes (to 256 nodes
 * with fsfem_set_deterministic).
 * nccl_unique_id == NULL with nranks > 1 gives a partition-only context: faces, assembly, BCs,
 * get_csr and spmv of rank r's rows work without any communicator; pcg_solve returns STATE.
 * Call before build_faces.  Errors: INVALID_ARG, STATE, NCCL. */
fsfem_status fsfem_comm_init(fsfem_ctx* ctx, const void* nccl_unique_id, int rank, int nranks);
/* Loopback group (SURVEY.md §4 "simulated partition"): ctxs[0..nranks) become ranks 0..nranks-1 of
 * ONE process, on one device and one stream (all created with the same cuda_device and
 * cuda_stream).  Each rank's faces, assembly and BCs are called on its own context as with NCCL;
 * fsfem_pcg_solve on any context of the group then runs the solve of every rank, with each
 * collective of the NCCL path (all-gather of partials, all-gather(v) or halo exchange of the
 * search direction, deterministic chunk partials) replaced by device-to-device copies on that
 * stream -- the multi-rank code path on one GPU.  The contexts stay owned by the caller (destroy
 * every one).  Call before build_faces.  Errors: INVALID_ARG (NULL, duplicates, different
 * device/stream), STATE. */
fsfem_status fsfem_comm_init_loopback(fsfem_ctx** ctxs, int nranks);
/* Node ranges of the ranks after build_faces: ranges [host, nranks + 1].  Errors: STATE. */
fsfem_status fsfem_get_partition(const fsfem_ctx* ctx, int64_t* ranges);
/* Deterministic dots (SURVEY.md 8(e) "Deterministic option"): every dot product of the solve is
 * a sum of per-chunk partials over fixed global chunks of 256 nodes, exchanged and summed in
 * chunk order; the SpMV runs in a canonical (partition-independent) order.  The displacements
 * are then bit-identical for any number of ranks (at some cost in speed).  Uses the standard
 * recurrence.  Set before build_faces (the ranges are aligned to the chunks); every rank must
 * agree.  Errors: STATE. */
fsfem_status fsfem_set_deterministic(fsfem_ctx* ctx, int on);
/* Rank 0 helper: write a fresh 128-byte ncclUniqueId to out [host].  Needs libnccl.so.2
 * (resolved at run time).  Errors: INVALID_ARG (NULL), NCCL. */
fsfem_status fsfem_nccl_get_unique_id(void* out);

/* Exchange of the search direction between ranks before each SpMV.
 * FSFEM_EXCHANGE_ALLGATHER (default): ncclAllGather of every rank's slice (8 * 3 N_n bytes).
 * FSFEM_EXCHANGE_HALO: each rank receives only its halo -- the columns of its rows owned by other
 * ranks (fsfem_get_halo) -- with ncclSend/ncclRecv, the sizes agreed once per mesh at the first
 * assemble_csr; remote entries outside the halo are never read.  The final solution is still
 * all-gathered.  Set before the first assemble_csr of a mesh.  Errors: INVALID_ARG, STATE,
 * NCCL (send/recv unavailable). */
enum { FSFEM_EXCHANGE_ALLGATHER = 0, FSFEM_EXCHANGE_HALO = 1 };
fsfem_status fsfem_set_exchange(fsfem_ctx* ctx, int mode);
/* Overlap (default off until measured on several GPUs): each PCG SpMV is split
 * into the chunks whose columns are all own rows and the others; the exchange of the search
 * direction (all-gather(v) or halo send/recv) runs on a side stream while the first part is
 * multiplied, and the second part waits for it (fork/join events, captured into the graphs).
 * Multi-rank, not with deterministic dots; uses the gather SpMV kernel.  Errors: none. */
fsfem_status fsfem_set_overlap(fsfem_ctx* ctx, int on);
/* The rank's halo after assemble_csr: *n = number of nodes (0 with one rank); nodes (host or
 * device, may be NULL) receives their global ids, ascending (so grouped by owner rank).  Works
 * on partition-only contexts.  Errors: STATE. */
fsfem_status fsfem_get_halo(const fsfem_ctx* ctx, int32_t* nodes, int64_t* n);

/* Discretisation of the stiffness (default FSFEM_METHOD_FS).  FSFEM_METHOD_FEM_T4 assembles the
 * conventional linear-tet stiffness K_e = V_e B^T c B over the tet node graph instead (the paper's
 * comparison column, PAPER.md:531 and Table 4 at 598-607); faces, BCs, SpMV
 * and PCG are shared.  Changing the method drops the assembled matrix (stage returns to "faces
 * built"); the next fsfem_assemble_csr rebuilds the pattern.  Errors: INVALID_ARG. */
typedef enum { FSFEM_METHOD_FS = 0, FSFEM_METHOD_FEM_T4 = 1 } fsfem_method;
fsfem_status fsfem_set_method(fsfem_ctx* ctx, int method);

/* Internal node order.  The SpMV and the assembly gather through L1/L2 and need a
 * banded numbering; mode 0 (default, auto) renumbers the nodes internally in Morton order of their
 * coordinates when the mean tet id span exceeds 16 N^(2/3), mode 1 always, mode 2 never.  Every
 * input and output of the API stays in the caller's numbering (faces, CSR rows and columns, loads,
 * Dirichlet ids, u, nodal stresses); only the internal storage order changes.  Single rank only
 * (with several ranks the row partition is in the caller's numbering).  Takes effect at the next
 * fsfem_build_faces.  Errors: INVALID_ARG. */
fsfem_status fsfem_set_reorder(fsfem_ctx* ctx, int mode);

/* PCG recurrence (default FSFEM_PCG_AUTO = the standard recurrence; the single-reduction form is
 * opt-in until the multi-GPU variants are measured).  FSFEM_PCG_STANDARD is the recurrence of the
 * oracle.  FSFEM_PCG_SINGLE_REDUCTION runs the
 * Chronopoulos-Gear form of the same Jacobi-PCG: s = K p is carried as a
 * vector, so each iteration has one SpMV (w = K u, u = D^-1 r) and ONE combined reduction of
 * (u.w, r.u, r.r) instead of two -- one collective per iteration on several GPUs.  Same
 * stopping test (||r|| <= rel_tol ||f||); rounding differs from the standard form, so iteration
 * counts may differ by a few percent.  Takes effect at the next pcg_solve.  Errors: INVALID_ARG. */
enum { FSFEM_PCG_STANDARD = 0, FSFEM_PCG_SINGLE_REDUCTION = 1, FSFEM_PCG_AUTO = 2 };
fsfem_status fsfem_set_pcg_variant(fsfem_ctx* ctx, int variant);

/* PCG loop control.  FSFEM_LOOP_DEVICE: the whole solve is ONE CUDA-graph launch whose while
 * node repeats a body of 8 iterations until the device-side recurrence stops -- no host
 * synchronisation inside the solve.  FSFEM_LOOP_HOST: graph batches of 32 iterations, the host
 * polls the state between batches (always used with NCCL ranks).  These two give bitwise
 * identical results at the same measured speed.  FSFEM_LOOP_CLUSTER: the whole
 * recurrence in ONE kernel launch on one thread-block cluster (up to 16 CTAs, reductions over
 * distributed shared memory, cluster barriers between the steps) -- for small meshes, where the
 * multi-kernel loop is launch-bound; single rank, standard recurrence, non-deterministic mode
 * only (otherwise the host loop runs).  Its reductions are grouped differently, so its rounding
 * (and possibly the iteration count) differs slightly from the other two; it is itself bitwise
 * reproducible.  FSFEM_LOOP_AUTO (default): CLUSTER when applicable and the operator has at
 * most 8000 stored + transposed blocks (where it was measured faster: cfg1), HOST otherwise.  Errors: INVALID_ARG. */
enum { FSFEM_LOOP_DEVICE = 0, FSFEM_LOOP_HOST = 1, FSFEM_LOOP_CLUSTER = 2, FSFEM_LOOP_AUTO = 3 };
fsfem_status fsfem_set_loop(fsfem_ctx* ctx, int mode);

/* S1: extract the unique faces of the mesh.
 *   xyz  [3*n_nodes] double, node coordinates (x, y, z per node)            (Node matrix)
 *   tets [4*n_tets]  int32, 0-based node ids; face l of a tet is the face
 *        opposite its vertex l                                               (Element matrix)
 *   n_faces, n_interior [host] receive N_f = N_i + N_e and N_i.
 * The mesh is copied into the context.  Errors: INVALID_ARG, DEGENERATE, TOPOLOGY, UNSUPPORTED. */
fsfem_status fsfem_build_faces(fsfem_ctx* ctx, const double* xyz, int64_t n_nodes,
                               const int32_t* tets, int64_t n_tets,
                               int64_t* n_faces, int64_t* n_interior);
/* Copy out the face table (Face_in / Face_out of PAPER.md:317, Fig. 7), ascending by (a,b,c):
 *   face_nodes [3*N_f] (a < b < c), face_tet [2*N_f] (t0 < t1, t1 = -1 exterior),
 *   face_opp [2*N_f] (node of t_k opposite the face, -1 exterior).  Any pointer may be NULL. */
fsfem_status fsfem_get_faces(const fsfem_ctx* ctx, int32_t* face_nodes, int32_t* face_tet,
                             int32_t* face_opp);

/* S2-S6 (Eqs. 8-9, 403-449): assemble the smoothed stiffness for Young's
 * modulus E > 0 and Poisson ratio nu in (-1, 0.5).  The first call also builds the symbolic
 * pattern (S5).  Every entry K[3i+a, 3j+c] = sum over faces f containing both i and j in
 * their field, in ascending face order, of V_f * (B_i^T c B_j)[a][c].
 *   row_begin, n_rows, nnz [host]: this rank's first global row, its row count, its nnz. */
fsfem_status fsfem_assemble_csr(fsfem_ctx* ctx, double E, double nu, int64_t* row_begin,
                                int64_t* n_rows, int64_t* nnz);
/* Copy out this rank's CSR rows: row_ptr [n_rows+1] (0-based, int64), col_idx [nnz] (global
 * column ids, ascending per row), vals [nnz].  Any pointer may be NULL. */
fsfem_status fsfem_get_csr(const fsfem_ctx* ctx, int64_t* row_ptr, int32_t* col_idx, double* vals);

/* S7: clamp every dof of the nodes dirichlet_nodes[n_dirichlet]
 * (prescribed displacement 0) and take nodal loads loads[3*n_nodes] (forces per dof).
 *   mode 0 = MODIFY (default): zero the constrained rows and columns except the diagonal,
 *            f_r = 0 on constrained dofs;
 *   mode 1 = PENALTY: K_rr += alpha, alpha = penalty_scale * max_i K_ii (penalty_scale <= 0
 *            means 1e8).
 * Also extracts the Jacobi preconditioner 1/K_ii.  Modifies the context's K in place. */
fsfem_status fsfem_apply_bc(fsfem_ctx* ctx, const int32_t* dirichlet_nodes, int64_t n_dirichlet,
                            const double* loads, int mode, double penalty_scale);

/* S8-S9: solve K u = f by Jacobi-PCG, stopping when ||r||_2 <= rel_tol * ||f||_2 on the
 * recurrence residual (rel_tol <= 0 means 1e-10; max_iter <= 0 means max(1000, 20*sqrt(n))).
 * At exit the true residual t = ||f - K u|| / ||f|| is recomputed; success (FSFEM_OK,
 * rep.converged = 1) requires t <= max(rel_tol, floor), floor = rep.residual_floor = the
 * fp64 rounding floor 2^-52 ||K||_F ||u|| / ||f|| (two PCGs stopped at 1e-10
 * cannot be asked for a true residual below the rounding of K u).  If the recurrence converged but
 * t misses, the solve restarts from u with r = f - K u (residual replacement, at most 2 restarts,
 * within max_iter) and returns NOT_CONVERGED if t still misses.
 *   u [3*n_nodes]: in = initial guess unless u0_is_zero, out = solution (full vector on every
 *   rank).  rep [host] may be NULL.  NOT_CONVERGED still writes u and rep. */
fsfem_status fsfem_pcg_solve(fsfem_ctx* ctx, double* u, int u0_is_zero, double rel_tol,
                             int64_t max_iter, fsfem_report* rep);

/* Strain / stress recovery ("first obtain the nodal displacements and then the
 * strain and stress", 457).  For the displacements u [3*n_nodes] (full vector),
 * per smoothing domain k (FS: face, in face order; FEM-T4: tet) the smoothed strain
 * eps_k = B_k u (Eq. 2 with Eq. 4's B; Voigt xx, yy, zz, yz, xz, xy, engineering shear) ->
 * strain [6*n_domains], stress = c eps -> stress [6*n_domains]; per own node the volume-weighted
 * mean of the stress over the domains whose field holds the node -> node_stress [6*n_nodes] and
 * its von Mises value -> node_vm [n_nodes] (only this rank's nodes are written).  Any output may
 * be NULL; n_domains [host] receives N_f (FS) or N_t (FEM-T4).  Needs assemble_csr (uses its E,
 * nu).  Errors: STATE, INVALID_ARG. */
fsfem_status fsfem_recover_stress(fsfem_ctx* ctx, const double* u, double* strain, double* stress,
                                  double* node_stress, double* node_vm, int64_t* n_domains);

/* Debug export of the dense stiffness of smoothing domains (Eq. 9
 * summand V_k Bbar_k^T c Bbar_k with Bbar_k of Eq. 7, 15x15 for an interior face and 12x12 for an
 * exterior one, Eq. 12; FEM-T4: V_e B_e^T c B_e of a tet), computed on the
 * device with the assembly's own arithmetic (same s vectors and M-form blocks as fsfem_assemble_csr).
 *   ids [n, host]: domain ids -- face ids in fsfem_get_faces order (FS-FEM) or tet ids (FEM-T4);
 *   K [n*225, host]: row-major 15x15 per domain, row / column 3I+a for field position I (faces:
 *     face nodes a < b < c, then the opposite vertices of face_tet[0] and face_tet[1]; tets: the 4
 *     nodes in the caller's tet order) and component a; rows / columns of an absent position
 *     (exterior face: 5th, tet: 5th) are 0;
 *   field [n*5, host] (may be NULL): the field node ids in the caller's numbering, -1 absent.
 * Needs assemble_csr (uses its E, nu and method).  Errors: STATE, INVALID_ARG (null K or ids with
 * n > 0, n < 0, an id out of range). */
fsfem_status fsfem_domain_stiffness(fsfem_ctx* ctx, const int64_t* ids, int64_t n, double* K, int32_t* field);

/* Nodal loads of a surface traction ("the nodal load is calculated"; 496-499: the
 * §4.1 beam's uniform pressure on its upper face).  node_flag [n_nodes] (bytes,
 * nonzero = on the loaded surface), traction [3, host] in N/m^2: every exterior face whose three
 * nodes are flagged gives each of them traction * area / 3.  loads [3*n_nodes] receives this rank's
 * node rows (others untouched).  Needs assemble_csr (uses its node lists).  The fixed mask of a
 * previous apply_bc is overwritten (apply_bc rebuilds it).  Errors: STATE, INVALID_ARG. */
fsfem_status fsfem_surface_loads(fsfem_ctx* ctx, const uint8_t* node_flag, const double* traction, double* loads);

/* Report of the last calls (timings and last PCG data); rep [host]. */
fsfem_status fsfem_get_report(const fsfem_ctx* ctx, fsfem_report* rep);

/* q = K p on the assembled matrix (before or after BCs): p [3*n_nodes], q [3*n_nodes] (this
 * rank's rows are written).  Used by tests for residual checks. */
fsfem_status fsfem_spmv(fsfem_ctx* ctx, const double* p, double* q);

#ifdef __cplusplus
}
#endif
#endif /* FSFEM_H */
