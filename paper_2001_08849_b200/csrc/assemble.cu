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

// Assembly record of a face (FS) or tet (FEM-T4), 144 bytes = 9 x 16 B:
//   doubles [0, 15): s_K for the 5 field nodes K (tets: 4; the 5th zero);
//   bytes [120, 140): int32 field node ids (a, b, c, opp0, opp1) (tets: 4 nodes, -1); 4 B pad.
// The domain volumes V_k live in a separate array (strain recovery).
constexpr int kRec = 18;  // doubles per record
__device__ __forceinline__ const int32_t* rec_field(const double* rec) {
  return reinterpret_cast<const int32_t*>(rec + 15);
}

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
                                                double* __restrict__ face_s, double* __restrict__ face_V) {
  __shared__ __align__(16) double stage[256 * kRec];
  // uniform trip count per block (every thread reaches the __syncthreads)
  for (int64_t fb0 = blockIdx.x * (int64_t)blockDim.x; fb0 < nf; fb0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = fb0 + threadIdx.x;
    const bool valid = f < nf;
    const int64_t fc = valid ? f : fb0;  // inactive threads recompute face fb0 and write nothing extra
    int32_t fld[5] = {face_nodes[3 * fc], face_nodes[3 * fc + 1], face_nodes[3 * fc + 2], face_opp[2 * fc],
                      face_opp[2 * fc + 1]};
    const int32_t tt[2] = {face_tet[2 * fc], face_tet[2 * fc + 1]};
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
    // stage the record of each face of the block in shared memory, then store coalesced
    double* st = stage + kRec * threadIdx.x;
#pragma unroll
    for (int K = 0; K < 5; ++K) {
      st[3 * K] = g[K][0] * rs;
      st[3 * K + 1] = g[K][1] * rs;
      st[3 * K + 2] = g[K][2] * rs;
    }
    int32_t* sfld = reinterpret_cast<int32_t*>(st + 15);
#pragma unroll
    for (int K = 0; K < 5; ++K) sfld[K] = fld[K];
    sfld[5] = 0;
    if (valid) face_V[f] = Vf;
    __syncthreads();
    const int64_t fb = f - threadIdx.x;  // first face of this block-iteration
    const int nvalid = static_cast<int>(nf - fb < (int64_t)blockDim.x ? nf - fb : (int64_t)blockDim.x);
    double2* dst = reinterpret_cast<double2*>(face_s + kRec * fb);
    const double2* src = reinterpret_cast<const double2*>(stage);
    for (int k = threadIdx.x; k < nvalid * (kRec / 2); k += blockDim.x) dst[k] = src[k];
    __syncthreads();
  }
}

// FEM-T4 (PAPER.md:531 and Table 4's FEM-T4 column): per tet
// s_I = sqrt(V_e) grad N_I (I = 0..3), so that V_e (B_I^T c B_J) = lam M + mu M^T + mu tr(M) I
// with M = s_I s_J^T, exactly the M-form of the faces.  Same 144-byte record as the faces.
__global__ void __launch_bounds__(256) k_tet_s(const double* __restrict__ xyz, const int32_t* __restrict__ tets,
                                               int64_t nt, double* __restrict__ tet_s, double* __restrict__ tet_V) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = reinterpret_cast<const int4*>(tets)[t];
    double x0, y0, z0, x1, y1, z1, x2, y2, z2, x3, y3, z3;
    load3(xyz, v.x, x0, y0, z0);
    load3(xyz, v.y, x1, y1, z1);
    load3(xyz, v.z, x2, y2, z2);
    load3(xyz, v.w, x3, y3, z3);
    const double e1x = x1 - x0, e1y = y1 - y0, e1z = z1 - z0;
    const double e2x = x2 - x0, e2y = y2 - y0, e2z = z2 - z0;
    const double e3x = x3 - x0, e3y = y3 - y0, e3z = z3 - z0;
    double g[4][3];
    g[1][0] = e2y * e3z - e2z * e3y;
    g[1][1] = e2z * e3x - e2x * e3z;
    g[1][2] = e2x * e3y - e2y * e3x;
    g[2][0] = e3y * e1z - e3z * e1y;
    g[2][1] = e3z * e1x - e3x * e1z;
    g[2][2] = e3x * e1y - e3y * e1x;
    g[3][0] = e1y * e2z - e1z * e2y;
    g[3][1] = e1z * e2x - e1x * e2z;
    g[3][2] = e1x * e2y - e1y * e2x;
    const double det = e1x * g[1][0] + e1y * g[1][1] + e1z * g[1][2];
    const double V = fabs(det) * (1.0 / 6.0);
    const double sc = sqrt(V) / det;  // grad N_q = (cross product) / det
    double* out = tet_s + kRec * t;
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      const double a = g[1][h] * sc, b = g[2][h] * sc, c = g[3][h] * sc;
      out[3 * 1 + h] = a;
      out[3 * 2 + h] = b;
      out[3 * 3 + h] = c;
      out[h] = -(a + b + c);
    }
    out[12] = out[13] = out[14] = 0.0;
    int32_t* ofld = reinterpret_cast<int32_t*>(out + 15);
    ofld[0] = v.x;
    ofld[1] = v.y;
    ofld[2] = v.z;
    ofld[3] = v.w;
    ofld[4] = -1;
    ofld[5] = 0;
    tet_V[t] = V;
  }
}

// Generic path (rows with more than 32 stored blocks; none in the Kuhn beams): warp per own
// node i; lane = stored block slot (j >= i, or halo j < n_lo; pattern.cuh), in chunks of 32.
// For every face of F(i) in ascending order, lanes whose neighbour j is in the face's field add
// s_i s_j^T.
template <bool kTet>
__global__ void __launch_bounds__(256) k_assemble_rows(
    const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr, const int64_t* __restrict__ nf_ptr,
    const int32_t* __restrict__ nf_idx, const int32_t* __restrict__ face_nodes, const int32_t* __restrict__ face_opp,
    const double* __restrict__ face_s, int64_t n_lo, int64_t nloc, double lam, double mu, double* __restrict__ vals,
    int min_deg) {
  const int lane = threadIdx.x & 31;
  for (int64_t il = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; il < nloc;
       il += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t self = static_cast<int32_t>(n_lo + il);
    const int64_t P = node_ptr[il];
    const int deg = static_cast<int>(node_ptr[il + 1] - P);
    if (deg <= min_deg) continue;  // handled by k_assemble_rows2
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
        const double* sf = face_s + kRec * static_cast<int64_t>(f);
        const int32_t* rf = rec_field(sf);
        const int32_t fld[5] = {rf[0], rf[1], rf[2], rf[3], rf[4]};
        int pi = 0, pj = -1;
#pragma unroll
        for (int K = 0; K < 5; ++K) {
          pi = (fld[K] == self) ? K : pi;
          pj = (fld[K] == j) ? K : pj;
        }
        if (pj >= 0) {
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


// Fast path, warp per own node i with <= 32 stored blocks (diagonal + j > i + halo j < n_lo).
// Rounds of 32 records (faces of F(i), or tets for FEM-T4; ascending):
//   load: the warp copies the round's 32 records (144 B each) into shared memory with
//      coalesced 16-byte loads (9 warp instructions, each covering ~4 records), instead of
//      each lane gathering its own record piece by piece (the L1 wavefront bound);
//   A. lane = face: add s_i s_i^T to the lane's diagonal partial sum, and for every other field node
//      that is a stored column of row i record (slot, s_K) and set the face's bit in the slot's
//      mask (order-independent OR);
//   B. lane = stored slot: walk the mask bits in ascending face order and add s_i s_K^T.
// Summation order (fixed, independent of timing): off-diagonal blocks in ascending face id, or
// for rows with <= 16 stored blocks (the common case) ascending over the even then the odd
// positions of each 32-face round; the diagonal block as per-lane sums over faces lane,
// lane+32, ... then a fixed warp tree.
constexpr int kRowWarps = 4;
#ifndef FSFEM_ASM_MINB
#define FSFEM_ASM_MINB 6
#endif
constexpr int kMaxTargets = 4;  // other field nodes of a face

template <bool kTet>
__global__ void __launch_bounds__(kRowWarps * 32, FSFEM_ASM_MINB) k_assemble_rows2(
    const int64_t* __restrict__ sptr, const int32_t* __restrict__ snbr, const int64_t* __restrict__ nf_ptr,
    const int32_t* __restrict__ nf_idx, const int32_t* __restrict__ face_nodes, const int32_t* __restrict__ face_opp,
    const double* __restrict__ face_s, int64_t n_lo, int64_t nloc, double lam, double mu, double* __restrict__ vals) {
  __shared__ __align__(16) double sh_rec[kRowWarps][32][kRec];
  __shared__ int32_t sh_cols[kRowWarps][32];
  __shared__ unsigned sh_mask[kRowWarps][32];
  __shared__ int8_t sh_pi[kRowWarps][32];
  __shared__ int8_t sh_tslot[kRowWarps][32][kMaxTargets];
  __shared__ int8_t sh_tk[kRowWarps][32][kMaxTargets];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t il = blockIdx.x * (int64_t)kRowWarps + w; il < nloc; il += (int64_t)gridDim.x * kRowWarps) {
    const int32_t self = static_cast<int32_t>(n_lo + il);
    const int64_t P = sptr[il];
    const int ds = static_cast<int>(sptr[il + 1] - P);
    if (ds > 32) continue;  // generic path
    const bool split = ds <= 16;
    sh_cols[w][lane] = lane < ds ? snbr[P + lane] : 0x7fffffff;
    sh_mask[w][lane] = 0u;
    const int64_t f0 = nf_ptr[il];
    const int nfc = static_cast<int>(nf_ptr[il + 1] - f0);
    double d[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // diagonal partial: xx yy zz xy xz yz
    double M[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) M[q] = 0.0;
    __syncwarp();
    for (int rb = 0; rb < nfc; rb += 32) {
      // ---- load the round's records: chunk c = 16-byte piece (c % 9) of record (c / 9)
      const int nact = min(32, nfc - rb);
      const int32_t myr = lane < nact ? nf_idx[f0 + rb + lane] : 0;
      // 16-byte cp.async (LDGSTS): global -> shared without registers, all 9 in flight
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int c = lane + 32 * q;
        const int k = c / 9, part = c - 9 * k;
        const int32_t r = __shfl_sync(0xffffffffu, myr, k);
        if (k < nact) {
          const double2* src = reinterpret_cast<const double2*>(face_s + kRec * static_cast<int64_t>(r)) + part;
          const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&sh_rec[w][0][0])) + 16u * c;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      // ---- A: lane = face
      if (lane < nact) {
        const double* sf = sh_rec[w][lane];
        const int32_t* rf = rec_field(sf);
        int32_t fld[5];
#pragma unroll
        for (int K = 0; K < 5; ++K) fld[K] = rf[K];
        int pi = 0;
#pragma unroll
        for (int K = 0; K < 5; ++K) pi = (fld[K] == self) ? K : pi;
        const double s0 = sf[3 * pi], s1 = sf[3 * pi + 1], s2 = sf[3 * pi + 2];
        sh_pi[w][lane] = static_cast<int8_t>(pi);
        d[0] = fma(s0, s0, d[0]);
        d[1] = fma(s1, s1, d[1]);
        d[2] = fma(s2, s2, d[2]);
        d[3] = fma(s0, s1, d[3]);
        d[4] = fma(s0, s2, d[4]);
        d[5] = fma(s1, s2, d[5]);
        int t = 0;
#pragma unroll
        for (int K = 0; K < 5; ++K) {
          const int32_t v = fld[K];
          if (K == pi || v < 0 || (v < self && v >= n_lo)) continue;
          // binary search of v in the stored columns (ascending, padded with INT_MAX)
          int lo = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1)
            if (sh_cols[w][lo + step - 1] < v) lo += step;
          sh_tslot[w][lane][t] = static_cast<int8_t>(lo);
          sh_tk[w][lane][t] = static_cast<int8_t>(K);
          atomicOr(&sh_mask[w][lo], 1u << lane);
          ++t;
        }
        for (; t < kMaxTargets; ++t) sh_tslot[w][lane][t] = -1;
      }
      __syncwarp();
      // ---- B: lane = stored slot; rows with <= 16 stored blocks give every slot 2 lanes, one for
      // the even and one for the odd record positions (combined at the end in that order)
      const int slot = split ? (lane & 15) : lane;
      unsigned m = sh_mask[w][slot];
      if (split) m &= (lane < 16) ? 0x55555555u : 0xAAAAAAAAu;
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        int t = 0;
#pragma unroll
        for (int q = 1; q < kMaxTargets; ++q) t = (sh_tslot[w][b][q] == slot) ? q : t;
        const double* rb_ = sh_rec[w][b];
        const int pb = sh_pi[w][b], K = sh_tk[w][b][t];
        const double a0 = rb_[3 * pb], a1 = rb_[3 * pb + 1], a2 = rb_[3 * pb + 2];
        const double c0 = rb_[3 * K], c1 = rb_[3 * K + 1], c2 = rb_[3 * K + 2];
        M[0] = fma(a0, c0, M[0]);
        M[1] = fma(a0, c1, M[1]);
        M[2] = fma(a0, c2, M[2]);
        M[3] = fma(a1, c0, M[3]);
        M[4] = fma(a1, c1, M[4]);
        M[5] = fma(a1, c2, M[5]);
        M[6] = fma(a2, c0, M[6]);
        M[7] = fma(a2, c1, M[7]);
        M[8] = fma(a2, c2, M[8]);
      }
      __syncwarp();
      sh_mask[w][lane] = 0u;
      __syncwarp();
    }
    if (split) {  // slot s = (even records) + (odd records): lane s adds lane s+16's partial
#pragma unroll
      for (int q = 0; q < 9; ++q) M[q] += __shfl_down_sync(0xffffffffu, M[q], 16);
    }
    // diagonal block: fixed warp tree of the per-lane partial sums
#pragma unroll
    for (int q = 0; q < 6; ++q) d[q] = warp_sum(d[q]);
    double* blocks = vals + 9 * P;
    const int32_t my_col = sh_cols[w][lane];
    if (lane < ds && my_col == self) {
      const double Md[9] = {d[0], d[3], d[4], d[3], d[1], d[5], d[4], d[5], d[2]};
#pragma unroll
      for (int q = 0; q < 9; ++q) M[q] = Md[q];
    }
    if (lane < ds) {
      const double tr = M[0] + M[4] + M[8];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double v = fma(lam, M[3 * a + c], mu * M[3 * c + a]);
          if (a == c) v = fma(mu, tr, v);
          blocks[9 * lane + 3 * a + c] = v;
        }
    }
    __syncwarp();
  }
}
}  // namespace

void face_s_device(const double* xyz, const int32_t* tets, const int32_t* face_nodes, const int32_t* face_tet,
                   const int32_t* face_opp, int64_t nf, double* face_s, double* face_V, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nf, 256), 16LL * num_sms()));
  k_face_s<<<std::max(grid, 1), 256, 0, s>>>(xyz, tets, face_nodes, face_tet, face_opp, nf, face_s, face_V);
  FS_LAUNCH_CHECK();
}

// rec_a/rec_b: FS (kTet = false) face_nodes/face_opp; FEM-T4 (tet = true) tets/unused.
void assemble_rows_device(const int64_t* node_ptr, const int32_t* nbr, const int64_t* nf_ptr, const int32_t* nf_idx,
                          const int32_t* face_nodes, const int32_t* face_opp, const double* face_s, int64_t n_lo,
                          int64_t nloc, double lam, double mu, double* vals, int64_t max_row_blocks, bool tet,
                          cudaStream_t s) {
  if (nloc == 0) return;
  // Persistent grid of exactly the resident CTAs: warp w takes nodes w, w + W, ... so the nodes in
  // flight form one contiguous window that slides forward; the field nodes of a face (which span
  // less than two windows in a banded numbering) are then assembled close together in time and
  // the face's record is re-read from L2, not DRAM.
  auto k2 = tet ? k_assemble_rows2<true> : k_assemble_rows2<false>;
  static int per_sm[2] = {0, 0};
  if (per_sm[tet] == 0) FS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[tet], k2, kRowWarps * 32, 0));
  const int g2 = static_cast<int>(
      std::min<int64_t>(ceil_div(nloc, kRowWarps), static_cast<int64_t>(std::max(1, per_sm[tet])) * num_sms()));
  k2<<<std::max(g2, 1), kRowWarps * 32, 0, s>>>(node_ptr, nbr, nf_ptr, nf_idx, face_nodes, face_opp, face_s, n_lo, nloc,
                                                lam, mu, vals);
  FS_LAUNCH_CHECK();
  if (max_row_blocks > 32) {
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nloc * 32, 256), 32LL * num_sms()));
    auto k1 = tet ? k_assemble_rows<true> : k_assemble_rows<false>;
    k1<<<std::max(grid, 1), 256, 0, s>>>(node_ptr, nbr, nf_ptr, nf_idx, face_nodes, face_opp, face_s, n_lo, nloc, lam,
                                         mu, vals, 32);
    FS_LAUNCH_CHECK();
  }
}

void tet_s_device(const double* xyz, const int32_t* tets, int64_t nt, double* tet_s, double* tet_V, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nt, 256), 16LL * num_sms()));
  k_tet_s<<<std::max(grid, 1), 256, 0, s>>>(xyz, tets, nt, tet_s, tet_V);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
