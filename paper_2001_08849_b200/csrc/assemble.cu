// S2-S4, S6 — per-face smoothed gradients and deterministic numeric assembly.
//
// Paper (Eqs. 7-9): for face k with smoothing domain Omega_k,
//     b_Ih = (1/V_k) sum_i n_ih N_I(x_i^G) A_i,   K = sum_k B_k^T c B_k V_k.
// The boundary integral of Eq. 7 is the divergence of the piecewise-linear N_I over the
// 1-2 cones (face, centroid of tet e), each of volume V_e/4 on which grad N_I = grad N_I^e;
// so (proved in SURVEY.md 8(c)):
//     V_k b_I = sum_{e ni k} (V_e/4) grad N_I^e,      V_k = sum_{e ni k} V_e/4.
// With w_I^e = (V_e/4) grad N_I^e = sign(det_e) * (cross product of two edges)/24 no division
// is needed per tet.  We keep s_I = (V_k b_I) / sqrt(V_k) per field node, so that
//     V_k (B_I^T c B_J)[a][c] = lambda M[a][c] + mu M[c][a] + mu delta_ac tr(M),
//     M = s_I s_J^T                                    (isotropic c, Voigt order of Eq. 4)
// and the global block K_IJ = lambda M_IJ + mu M_IJ^T + mu tr(M_IJ) I with
// M_IJ = sum over faces holding I and J of s_I s_J^T, summed in ascending face id.
#include "common.cuh"

namespace fsfem {

namespace {

constexpr int kFaceStride = 16;  // doubles per face: 5 field nodes x 3 + V_f

__device__ __forceinline__ void load3(const double* __restrict__ xyz, int32_t v, double& x, double& y, double& z) {
  x = xyz[3 * v];
  y = xyz[3 * v + 1];
  z = xyz[3 * v + 2];
}

// Thread per face: s_K for the field nodes K = (a, b, c, d, e) of face f.
__global__ void __launch_bounds__(256) k_face_s(const double* __restrict__ xyz, const int32_t* __restrict__ tets,
                                                const int32_t* __restrict__ face_nodes,
                                                const int32_t* __restrict__ face_tet,
                                                const int32_t* __restrict__ face_opp, int64_t nf,
                                                double* __restrict__ face_s) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    int32_t fld[5] = {face_nodes[3 * f], face_nodes[3 * f + 1], face_nodes[3 * f + 2], face_opp[2 * f],
                      face_opp[2 * f + 1]};
    const int32_t tt[2] = {face_tet[2 * f], face_tet[2 * f + 1]};
    double g[5][3];
#pragma unroll
    for (int K = 0; K < 5; ++K) g[K][0] = g[K][1] = g[K][2] = 0.0;
    double Vf = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int32_t t = tt[e];
      if (t < 0) continue;
      const int4 v = reinterpret_cast<const int4*>(tets)[t];
      const int32_t vid[4] = {v.x, v.y, v.z, v.w};
      double x0, y0, z0, x1, y1, z1, x2, y2, z2, x3, y3, z3;
      load3(xyz, v.x, x0, y0, z0);
      load3(xyz, v.y, x1, y1, z1);
      load3(xyz, v.z, x2, y2, z2);
      load3(xyz, v.w, x3, y3, z3);
      const double e1x = x1 - x0, e1y = y1 - y0, e1z = z1 - z0;
      const double e2x = x2 - x0, e2y = y2 - y0, e2z = z2 - z0;
      const double e3x = x3 - x0, e3y = y3 - y0, e3z = z3 - z0;
      // c1 = e2 x e3, c2 = e3 x e1, c3 = e1 x e2 ; det = e1 . c1
      double w[4][3];
      w[1][0] = e2y * e3z - e2z * e3y;
      w[1][1] = e2z * e3x - e2x * e3z;
      w[1][2] = e2x * e3y - e2y * e3x;
      w[2][0] = e3y * e1z - e3z * e1y;
      w[2][1] = e3z * e1x - e3x * e1z;
      w[2][2] = e3x * e1y - e3y * e1x;
      w[3][0] = e1y * e2z - e1z * e2y;
      w[3][1] = e1z * e2x - e1x * e2z;
      w[3][2] = e1x * e2y - e1y * e2x;
      const double det = e1x * w[1][0] + e1y * w[1][1] + e1z * w[1][2];
      const double sc = (det > 0.0 ? 1.0 : -1.0) * (1.0 / 24.0);
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        w[1][h] *= sc;
        w[2][h] *= sc;
        w[3][h] *= sc;
        w[0][h] = -(w[1][h] + w[2][h] + w[3][h]);
      }
      Vf += fabs(det) * (1.0 / 24.0);
      // scatter the tet's 4 vertex weights onto the field positions
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int K = 0; K < 5; ++K) {
          if (fld[K] == vid[q]) {
            g[K][0] += w[q][0];
            g[K][1] += w[q][1];
            g[K][2] += w[q][2];
          }
        }
      }
    }
    const double rs = 1.0 / sqrt(Vf);
    double* out = face_s + kFaceStride * f;
#pragma unroll
    for (int K = 0; K < 5; ++K) {
      out[3 * K] = g[K][0] * rs;
      out[3 * K + 1] = g[K][1] * rs;
      out[3 * K + 2] = g[K][2] * rs;
    }
    out[15] = Vf;
  }
}

// Warp per own node i; lane = stored block slot (j >= i, or halo j < n_lo; pattern.cuh), in
// chunks of 32.  For every face of F(i) in ascending order, lanes whose neighbour j is in the
// face's field add s_i s_j^T.
__global__ void __launch_bounds__(256) k_assemble_rows(
    const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr, const int64_t* __restrict__ nf_ptr,
    const int32_t* __restrict__ nf_idx, const int32_t* __restrict__ face_nodes, const int32_t* __restrict__ face_opp,
    const double* __restrict__ face_s, int64_t n_lo, int64_t nloc, double lam, double mu, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  for (int64_t il = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; il < nloc;
       il += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t self = static_cast<int32_t>(n_lo + il);
    const int64_t P = node_ptr[il];
    const int deg = static_cast<int>(node_ptr[il + 1] - P);
    const int64_t f0 = nf_ptr[il], f1 = nf_ptr[il + 1];
    double* blocks = vals + 9 * P;
    for (int s0 = 0; s0 < deg; s0 += 32) {
      const int s = s0 + lane;
      const int32_t j = (s < deg) ? nbr[P + s] : -2;
      double M[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) M[q] = 0.0;
      for (int64_t k = f0; k < f1; ++k) {
        const int32_t f = nf_idx[k];
        const int32_t fld[5] = {face_nodes[3 * f], face_nodes[3 * f + 1], face_nodes[3 * f + 2], face_opp[2 * f],
                                face_opp[2 * f + 1]};
        int pi = 0, pj = -1;
#pragma unroll
        for (int K = 0; K < 5; ++K) {
          pi = (fld[K] == self) ? K : pi;
          pj = (fld[K] == j) ? K : pj;
        }
        if (pj >= 0) {
          const double* sf = face_s + kFaceStride * f;
          const double si0 = sf[3 * pi], si1 = sf[3 * pi + 1], si2 = sf[3 * pi + 2];
          const double sj0 = sf[3 * pj], sj1 = sf[3 * pj + 1], sj2 = sf[3 * pj + 2];
          M[0] = fma(si0, sj0, M[0]);
          M[1] = fma(si0, sj1, M[1]);
          M[2] = fma(si0, sj2, M[2]);
          M[3] = fma(si1, sj0, M[3]);
          M[4] = fma(si1, sj1, M[4]);
          M[5] = fma(si1, sj2, M[5]);
          M[6] = fma(si2, sj0, M[6]);
          M[7] = fma(si2, sj1, M[7]);
          M[8] = fma(si2, sj2, M[8]);
        }
      }
      if (s < deg) {
        const double tr = M[0] + M[4] + M[8];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double v = fma(lam, M[3 * a + c], mu * M[3 * c + a]);
            if (a == c) v = fma(mu, tr, v);
            blocks[9 * s + 3 * a + c] = v;
          }
      }
    }
  }
}

}  // namespace

void face_s_device(const double* xyz, const int32_t* tets, const int32_t* face_nodes, const int32_t* face_tet,
                   const int32_t* face_opp, int64_t nf, double* face_s, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nf, 256), 16LL * num_sms()));
  k_face_s<<<std::max(grid, 1), 256, 0, s>>>(xyz, tets, face_nodes, face_tet, face_opp, nf, face_s);
  FS_LAUNCH_CHECK();
}

void assemble_rows_device(const int64_t* node_ptr, const int32_t* nbr, const int64_t* nf_ptr, const int32_t* nf_idx,
                          const int32_t* face_nodes, const int32_t* face_opp, const double* face_s, int64_t n_lo,
                          int64_t nloc, double lam, double mu, double* vals, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nloc * 32, 256), 32LL * num_sms()));
  k_assemble_rows<<<std::max(grid, 1), 256, 0, s>>>(node_ptr, nbr, nf_ptr, nf_idx, face_nodes, face_opp, face_s, n_lo,
                                                    nloc, lam, mu, vals);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
