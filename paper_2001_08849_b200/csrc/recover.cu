// Smoothed strain / stress recovery ("first obtain the nodal
// displacements and then the strain and stress", 457).
//
// Per smoothing domain k (FS: face; FEM-T4: tet) the strain of Eq. 2 with the B-bar of Eq. 4,
//     eps_k = sum_I B_I u_I   (Voigt xx, yy, zz, yz, xz, xy; engineering shear),
// from the assembly records (face_s / tet_s: s_I = sqrt(V_k) b_I and V_k), and
//     sigma_k = lam tr(eps) [1 1 1 0 0 0] + mu diag(2 2 2 1 1 1) eps        (isotropic c, Q1).
// Per own node the volume-weighted mean of sigma over the domains whose field holds the node
// (ascending domain id, the per-node lists of the assembly), and its von Mises value.
#include "common.cuh"

namespace fsfem {

namespace {

constexpr int kRecStride = 16;  // doubles per assembly record (assemble.cu): s_K at 3K

__device__ __forceinline__ void domain_field(const int32_t* __restrict__ rec_a, const int32_t* __restrict__ rec_b,
                                             bool tet, int64_t r, int32_t (&fld)[5]) {
  if (tet) {
    const int4 v = reinterpret_cast<const int4*>(rec_a)[r];
    fld[0] = v.x;
    fld[1] = v.y;
    fld[2] = v.z;
    fld[3] = v.w;
    fld[4] = -1;
  } else {
    fld[0] = rec_a[3 * r];
    fld[1] = rec_a[3 * r + 1];
    fld[2] = rec_a[3 * r + 2];
    fld[3] = rec_b[2 * r];
    fld[4] = rec_b[2 * r + 1];
  }
}

__global__ void __launch_bounds__(256) k_domain_stress(const int32_t* __restrict__ rec_a,
                                                       const int32_t* __restrict__ rec_b, bool tet,
                                                       const double* __restrict__ rec_s,
                                                       const double* __restrict__ rec_V, int64_t nrec,
                                                       const double* __restrict__ u, double lam, double mu,
                                                       double* __restrict__ strain, double* __restrict__ stress) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrec; r += (int64_t)gridDim.x * blockDim.x) {
    int32_t fld[5];
    domain_field(rec_a, rec_b, tet, r, fld);
    const double* sr = rec_s + kRecStride * r;
    const double V = rec_V[r];
    const double inv = 1.0 / sqrt(V);
    double e[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int K = 0; K < 5; ++K) {
      if (fld[K] < 0) continue;
      const double bx = sr[3 * K] * inv, by = sr[3 * K + 1] * inv, bz = sr[3 * K + 2] * inv;
      const double* uk = u + 3 * static_cast<int64_t>(fld[K]);
      const double ux = uk[0], uy = uk[1], uz = uk[2];
      e[0] = fma(bx, ux, e[0]);
      e[1] = fma(by, uy, e[1]);
      e[2] = fma(bz, uz, e[2]);
      e[3] = fma(bz, uy, fma(by, uz, e[3]));
      e[4] = fma(bz, ux, fma(bx, uz, e[4]));
      e[5] = fma(by, ux, fma(bx, uy, e[5]));
    }
    const double tr = e[0] + e[1] + e[2];
    const double s[6] = {fma(lam, tr, 2.0 * mu * e[0]), fma(lam, tr, 2.0 * mu * e[1]), fma(lam, tr, 2.0 * mu * e[2]),
                         mu * e[3], mu * e[4], mu * e[5]};
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (strain) strain[6 * r + q] = e[q];
      stress[6 * r + q] = s[q];
    }
  }
}

// Thread per own node: sum over its domain list in ascending order (fixed order).
__global__ void __launch_bounds__(256) k_node_stress(const int64_t* __restrict__ nd_ptr,
                                                     const int32_t* __restrict__ nd_idx, const double* __restrict__ rec_V,
                                                     const double* __restrict__ stress, int64_t nloc,
                                                     double* __restrict__ node_stress, double* __restrict__ node_vm) {
  for (int64_t il = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; il < nloc; il += (int64_t)gridDim.x * blockDim.x) {
    double a[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, w = 0.0;
    for (int64_t k = nd_ptr[il]; k < nd_ptr[il + 1]; ++k) {
      const int64_t r = nd_idx[k];
      const double V = rec_V[r];
#pragma unroll
      for (int q = 0; q < 6; ++q) a[q] = fma(V, stress[6 * r + q], a[q]);
      w += V;
    }
    const double iw = w > 0.0 ? 1.0 / w : 0.0;
#pragma unroll
    for (int q = 0; q < 6; ++q) a[q] *= iw;
    if (node_stress)
#pragma unroll
      for (int q = 0; q < 6; ++q) node_stress[6 * il + q] = a[q];
    if (node_vm) {
      const double d01 = a[0] - a[1], d12 = a[1] - a[2], d20 = a[2] - a[0];
      node_vm[il] = sqrt(0.5 * (d01 * d01 + d12 * d12 + d20 * d20) + 3.0 * (a[3] * a[3] + a[4] * a[4] + a[5] * a[5]));
    }
  }
}

}  // namespace

void recover_device(const int32_t* rec_a, const int32_t* rec_b, bool tet, const double* rec_s, const double* rec_V,
                    int64_t nrec,
                    const int64_t* nd_ptr, const int32_t* nd_idx, int64_t nloc, const double* u, double lam, double mu,
                    double* strain, double* stress, double* node_stress, double* node_vm, cudaStream_t s) {
  const int g1 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nrec, 256), 16LL * num_sms())));
  k_domain_stress<<<g1, 256, 0, s>>>(rec_a, rec_b, tet, rec_s, rec_V, nrec, u, lam, mu, strain, stress);
  FS_LAUNCH_CHECK();
  if (nloc > 0 && (node_stress || node_vm)) {
    const int g2 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 256), 16LL * num_sms())));
    k_node_stress<<<g2, 256, 0, s>>>(nd_ptr, nd_idx, rec_V, stress, nloc, node_stress, node_vm);
    FS_LAUNCH_CHECK();
  }
}

}  // namespace fsfem

// ---------------------------------------------------------------------------------------------
// Surface loads ("the nodal load is calculated"; 496-499: uniform pressure on the
// upper face): each exterior face whose three nodes are flagged gives each of
// them traction * A / 3.  Thread per own node, over its assembly list in ascending order
// (FS: the faces holding the node; FEM-T4: its tets, whose exterior faces are found through
// tet_face -- an exterior face has exactly one tet): deterministic, no atomics.
namespace fsfem {
namespace {

__device__ __forceinline__ double tri_area(const double* __restrict__ xyz, int32_t a, int32_t b, int32_t c) {
  const double ax = xyz[3 * a], ay = xyz[3 * a + 1], az = xyz[3 * a + 2];
  const double ux = xyz[3 * b] - ax, uy = xyz[3 * b + 1] - ay, uz = xyz[3 * b + 2] - az;
  const double vx = xyz[3 * c] - ax, vy = xyz[3 * c + 1] - ay, vz = xyz[3 * c + 2] - az;
  const double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
  return 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
}

__global__ void __launch_bounds__(256) k_surface_loads(const int64_t* __restrict__ nd_ptr,
                                                       const int32_t* __restrict__ nd_idx, bool tet,
                                                       const int32_t* __restrict__ tet_face,
                                                       const int32_t* __restrict__ face_nodes,
                                                       const int32_t* __restrict__ face_tet,
                                                       const uint8_t* __restrict__ flag,
                                                       const double* __restrict__ xyz, int64_t n_lo, int64_t nloc,
                                                       double tx, double ty, double tz, double* __restrict__ loads) {
  for (int64_t il = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; il < nloc; il += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = static_cast<int32_t>(n_lo + il);
    double A = 0.0;
    for (int64_t k = nd_ptr[il]; k < nd_ptr[il + 1]; ++k) {
      const int32_t r = nd_idx[k];
      const int nl = tet ? 4 : 1;
      for (int l = 0; l < nl; ++l) {
        const int32_t f = tet ? tet_face[4 * r + l] : r;
        if (face_tet[2 * f + 1] >= 0) continue;  // interior face
        const int32_t a = face_nodes[3 * f], b = face_nodes[3 * f + 1], c = face_nodes[3 * f + 2];
        if (a != i && b != i && c != i) continue;
        if (!flag[a] || !flag[b] || !flag[c]) continue;
        A += tri_area(xyz, a, b, c) * (1.0 / 3.0);
      }
    }
    loads[3 * il] = tx * A;
    loads[3 * il + 1] = ty * A;
    loads[3 * il + 2] = tz * A;
  }
}

}  // namespace

void surface_loads_device(const int64_t* nd_ptr, const int32_t* nd_idx, bool tet, const int32_t* tet_face,
                          const int32_t* face_nodes, const int32_t* face_tet, const uint8_t* flag, const double* xyz,
                          int64_t n_lo, int64_t nloc, const double* t, double* loads, cudaStream_t s) {
  if (nloc == 0) return;
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 256), 16LL * num_sms())));
  k_surface_loads<<<g, 256, 0, s>>>(nd_ptr, nd_idx, tet, tet_face, face_nodes, face_tet, flag, xyz, n_lo, nloc, t[0],
                                    t[1], t[2], loads);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
