/* FS-FEM CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 implementation of the FS-FEM hot path of
 * arxiv 2001.08849 (juSFEM), written from PAPER.md.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2001_08849_b200/csrc).
 *
 * Parity pins for every function live in tests/test_oracle_*.py (see DESIGN.md "Oracle
 * pins").  Nothing here is "parity unpinned".
 *
 * Status codes: 0 ok, 1 invalid argument, 2 topology (face shared by >2 tets),
 * 3 degenerate tet, 4 not converged, 5 breakdown, 6 state (call order).
 */
#ifndef FSFEM_ORACLE_H
#define FSFEM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct ora_mesh ora_mesh;

/* Copies xyz[3*nn] and tets[4*nt] (0-based).  Never fails except on allocation. */
ora_mesh* ora_new(const double* xyz, int64_t nn, const int32_t* tets, int64_t nt);
void ora_free(ora_mesh* m);
const char* ora_error(const ora_mesh* m);

/* O1 (Eq. 10): ids in range and distinct, |V| > 1e-14 * diag(bbox)^3.
 * vol_out[nt] (may be NULL) receives Eq. 10 (the signed 4x4 determinant / 6). */
int ora_validate(ora_mesh* m, double* vol_out);

/* O2 (Fig. 7, Alg. 1): face table from a std::map keyed by the sorted
 * vertex triple.  Faces ascending by (a,b,c); t0 < t1; exterior: t1 = opp1 = -1. */
int ora_build_faces(ora_mesh* m, int64_t* n_faces, int64_t* n_interior);
void ora_get_faces(const ora_mesh* m, int32_t* face_nodes, int32_t* face_tet, int32_t* face_opp);

/* O3/O4 for one face (Fig. 1, 195-226 Eq. 7 + Table 1):
 * field[5] = (a,b,c,d,e) (e = -1 exterior); bbar[5*3] = b_Ih; *Vf = smoothing-domain volume;
 * *P = number of boundary triangles (6 / 4); tri[P*9] = per triangle (A, n_x, n_y, n_z,
 * N_a, N_b, N_c, N_d, N_e) at its centroid. tri may be NULL. */
int ora_face_domain(ora_mesh* m, int64_t f, int32_t* field, double* bbar, double* Vf,
                    int* P, double* tri);

/* O4/O5 (Eqs. 8-9, 403-416 Eq. 12, 449 sparse()): dense K_f per face,
 * COO of all 9*n_f^2 entries, stable sort by (row, col) in emission order, summed.
 * Only rows of nodes in [node_lo, node_hi) are kept.  Structural zeros are kept. */
int ora_assemble_fs(ora_mesh* m, double E, double nu, int64_t node_lo, int64_t node_hi);
/* O8 (conventional FEM-T4): K_e = V_e B^T c B per tet, same COO->CSR. */
int ora_assemble_fem(ora_mesh* m, double E, double nu, int64_t node_lo, int64_t node_hi);
/* K7: dense stiffness of one smoothing domain -- face f (Eq. 9 summand
 * V_k Bbar^T c Bbar, 15x15 interior / 12x12 exterior) or, for FEM-T4,
 * tet t (V_e B^T c B) -- into K[15*15] row-major, row/column 3I+a for field position I
 * (faces: a, b, c, opp0, opp1; tets: the 4 nodes in tet order), absent positions zero;
 * field[5] = node ids, -1 absent. */
int ora_face_stiffness(ora_mesh* m, int64_t f, double E, double nu, double* K, int32_t* field);
int ora_tet_stiffness(ora_mesh* m, int64_t t, double E, double nu, double* K, int32_t* field);
/* Triplets emitted by the last ora_assemble_fs (Eq. 12: N_e*144 + N_i*225 for all rows). */
int64_t ora_last_coo_count(const ora_mesh* m);
/* Replace K by a caller CSR over all 3*nn rows (used by solver pins on hand-made matrices). */
int ora_set_csr(ora_mesh* m, int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx, const double* vals);
void ora_csr_dims(const ora_mesh* m, int64_t* row_lo, int64_t* n_rows, int64_t* nnz);
void ora_get_csr(const ora_mesh* m, int64_t* row_ptr, int32_t* col_idx, double* vals);
/* y = K x on the current (full) CSR; rows summed in column order. */
int ora_spmv(const ora_mesh* m, const double* x, double* y);

/* O6 (PAPER.md:243-245 STEP 5; 449 penalty): mode 0 MODIFY (zero constrained rows and
 * columns, keep K_rr, f_r = K_rr*g_r with g = 0), mode 1 PENALTY (K_rr += alpha,
 * alpha = scale * max_i K_ii, scale <= 0 -> 1e8).  loads[3*nn] -> f. */
int ora_apply_bc(ora_mesh* m, const int32_t* dirichlet, int64_t n_dir, const double* loads,
                 int mode, double penalty_scale);
void ora_get_rhs(const ora_mesh* m, double* f);

/* O7: Jacobi-PCG from x0 = 0, recurrence residual ||r||/||f|| <= tol. */
int ora_pcg(ora_mesh* m, double tol, int64_t max_iter, double* u, int64_t* iters,
            double* rel_res, double* true_rel_res);
/* O7: banded Cholesky L L^T of the (BC-applied) K, exact to rounding. */
int ora_cholesky(ora_mesh* m, double* u);
/* O6 check: exact elimination — Cholesky of K with constrained rows/cols removed, on the
 * current (unmodified, pre-BC) K; u_r = 0 on constrained dofs. */
int ora_cholesky_eliminate(ora_mesh* m, const int32_t* dirichlet, int64_t n_dir,
                           const double* loads, double* u);

/* O9: smoothed strain eps_k = B_k d (Eq. 2, 4) and stress
 * sigma_k = c eps_k per face [6*N_f] (Voigt xx,yy,zz,yz,xz,xy, engineering shear), the
 * volume-weighted nodal mean of sigma over the faces whose field holds the node [6*nn] and its von
 * Mises value [nn].  Any output may be NULL. */
int ora_recover(ora_mesh* m, double E, double nu, const double* u, double* strain, double* stress,
                double* node_stress, double* node_vm);

/* O10: nodal loads [3*nn] of a uniform traction[3] (N/m^2) on the exterior
 * faces whose 3 nodes all have node_flag[] != 0: each such node gets traction * A_face / 3. */
int ora_surface_loads(ora_mesh* m, const uint8_t* node_flag, const double* traction, double* loads);

#ifdef __cplusplus
}
#endif
#endif
