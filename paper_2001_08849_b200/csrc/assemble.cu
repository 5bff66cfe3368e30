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
#include "pattern.cuh"

namespace fsfem {

namespace {

// Assembly record of a face (FS) or tet (FEM-T4), 128 bytes = one line:
//   doubles [0, 15): s_K for the 5 field nodes K (tets: 4; the 5th zero); [15]: V_k.
// The field node ids are not stored: the assembly program (below) names them by position.
constexpr int kRec = 16;  // doubles per record

// Field nodes of record r: FS (a, b, c, opp0, opp1) from face_nodes / face_opp; FEM-T4 the
// 4 tet nodes and -1.
__device__ __forceinline__ void field_of(const int32_t* __restrict__ rec_a, const int32_t* __restrict__ rec_b,
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

__device__ __forceinline__ void load3(const double* __restrict__ xyz, int32_t v, double& x, double& y, double& z) {
  // (32-B padded coordinates with one 256-bit load per vertex were slower: 326 vs 291 us, cfg4)
  x = __ldg(xyz + 3 * (int64_t)v);
  y = __ldg(xyz + 3 * (int64_t)v + 1);
  z = __ldg(xyz + 3 * (int64_t)v + 2);
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
    // The two tets of the face are (a, b, c, d) and (a, b, c, e) with its field nodes
    // (a, b, c, d, e) = (face nodes, opposite vertices of face_tet[0], face_tet[1]): only 5 distinct
    // vertices, and each tet's vertex weights land on known field positions (no matching).  The
    // weights do not depend on the vertex order of the tet: the sign of det fixes the orientation.
    const int32_t na = face_nodes[3 * fc], nb = face_nodes[3 * fc + 1], nc = face_nodes[3 * fc + 2];
    const int32_t nd = face_opp[2 * fc], ne = face_opp[2 * fc + 1];
    double ax, ay, az, bx, by, bz, cx, cy, cz, dx, dy, dz;
    load3(xyz, na, ax, ay, az);
    load3(xyz, nb, bx, by, bz);
    load3(xyz, nc, cx, cy, cz);
    load3(xyz, nd, dx, dy, dz);
    double ex = 0.0, ey = 0.0, ez = 0.0;
    if (ne >= 0) load3(xyz, ne, ex, ey, ez);
    const double e1x = bx - ax, e1y = by - ay, e1z = bz - az;
    const double e2x = cx - ax, e2y = cy - ay, e2z = cz - az;
    // e1 x e2 is shared by both tets (weight of the opposite vertex, up to the tet's scale)
    const double c3x = e1y * e2z - e1z * e2y, c3y = e1z * e2x - e1x * e2z, c3z = e1x * e2y - e1y * e2x;
    double g[5][3];
    double Vf = 0.0;
    {  // tet (a, b, c, d)
      const double e3x = dx - ax, e3y = dy - ay, e3z = dz - az;
      const double c1x = e2y * e3z - e2z * e3y, c1y = e2z * e3x - e2x * e3z, c1z = e2x * e3y - e2y * e3x;
      const double c2x = e3y * e1z - e3z * e1y, c2y = e3z * e1x - e3x * e1z, c2z = e3x * e1y - e3y * e1x;
      const double det = e1x * c1x + e1y * c1y + e1z * c1z;
      const double sc = (det > 0.0 ? 1.0 : -1.0) * (1.0 / 24.0);
      g[1][0] = c1x * sc; g[1][1] = c1y * sc; g[1][2] = c1z * sc;
      g[2][0] = c2x * sc; g[2][1] = c2y * sc; g[2][2] = c2z * sc;
      g[3][0] = c3x * sc; g[3][1] = c3y * sc; g[3][2] = c3z * sc;
#pragma unroll
      for (int h = 0; h < 3; ++h) g[0][h] = -(g[1][h] + g[2][h] + g[3][h]);
      g[4][0] = g[4][1] = g[4][2] = 0.0;
      Vf = fabs(det) * (1.0 / 24.0);
    }
    if (ne >= 0) {  // tet (a, b, c, e)
      const double e3x = ex - ax, e3y = ey - ay, e3z = ez - az;
      const double c1x = e2y * e3z - e2z * e3y, c1y = e2z * e3x - e2x * e3z, c1z = e2x * e3y - e2y * e3x;
      const double c2x = e3y * e1z - e3z * e1y, c2y = e3z * e1x - e3x * e1z, c2z = e3x * e1y - e3y * e1x;
      const double det = e1x * c1x + e1y * c1y + e1z * c1z;
      const double sc = (det > 0.0 ? 1.0 : -1.0) * (1.0 / 24.0);
      const double w1[3] = {c1x * sc, c1y * sc, c1z * sc}, w2[3] = {c2x * sc, c2y * sc, c2z * sc},
                   w3[3] = {c3x * sc, c3y * sc, c3z * sc};
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        g[0][h] += -(w1[h] + w2[h] + w3[h]);
        g[1][h] += w1[h];
        g[2][h] += w2[h];
        g[4][h] = w3[h];
      }
      Vf += fabs(det) * (1.0 / 24.0);
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
    st[15] = Vf;
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
    out[15] = V;
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
        int32_t fld[5];
        field_of(face_nodes, face_opp, kTet, f, fld);
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


// Assembly program (once per pattern; thread per own node, faces of F(i) in ascending order):
// nf_pi[k] = field position of i in the k-th face; for every other field node v that is a
// stored column of row i (v > i, or a halo column v < n_lo) the entry k | (position of v) << 13
// is appended to the list of v's stored block, so every list is ascending in k.
constexpr int kProgMaxFaces = 8000;  // k < 8192 - 32 keeps the 0xffff sentinel above every round

// Warp per own node; the faces of F(i) in rounds of 32 (lane = face).  Count pass: nf_pi and the
// number of entries of every stored block (shared counters; order irrelevant).  Fill pass: per
// round, slot by slot, the lanes holding the slot's column write in lane (= ascending face) order.
constexpr int kProgWarps = 8;
template <bool kFill>
__global__ void __launch_bounds__(kProgWarps * 32) k_prog(
    const int64_t* __restrict__ sptr, const int32_t* __restrict__ snbr, const int64_t* __restrict__ nf_ptr,
    const int32_t* __restrict__ nf_idx, const int32_t* __restrict__ rec_a, const int32_t* __restrict__ rec_b, bool tet,
    int64_t n_lo, int64_t nloc, uint8_t* __restrict__ nf_pi, int32_t* __restrict__ cnt,
    const int32_t* __restrict__ blk_ent, uint16_t* __restrict__ prog, unsigned long long* __restrict__ err) {
  __shared__ int32_t sh_cols[kProgWarps][32];
  __shared__ int32_t sh_cnt[kProgWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t il = blockIdx.x * (int64_t)kProgWarps + w; il < nloc; il += (int64_t)gridDim.x * kProgWarps) {
    const int32_t i = static_cast<int32_t>(n_lo + il);
    const int64_t P = sptr[il];
    const int ds = static_cast<int>(sptr[il + 1] - P);
    if (ds > 32) continue;  // generic path (no program)
    const int64_t f0 = nf_ptr[il];
    const int nfc = static_cast<int>(nf_ptr[il + 1] - f0);
    if (nfc >= kProgMaxFaces) {
      if (!kFill && lane == 0) report_error(err, FSFEM_ERR_UNSUPPORTED, i);
      continue;
    }
    sh_cols[w][lane] = lane < ds ? snbr[P + lane] : 0x7fffffff;
    sh_cnt[w][lane] = (kFill && lane < ds) ? blk_ent[P + lane] : 0;
    __syncwarp();
    for (int rb = 0; rb < nfc; rb += 32) {
      const int k = rb + lane;
      int tslot[4] = {-1, -1, -1, -1}, tk[4] = {0, 0, 0, 0};
      if (k < nfc) {
        int32_t fld[5];
        field_of(rec_a, rec_b, tet, nf_idx[f0 + k], fld);
        int pi = 0;
#pragma unroll
        for (int K = 0; K < 5; ++K) pi = (fld[K] == i) ? K : pi;
        if (!kFill) nf_pi[f0 + k] = static_cast<uint8_t>(pi);
        int t = 0;
#pragma unroll
        for (int K = 0; K < 5; ++K) {
          const int32_t v = fld[K];
          if (K == pi || v < 0 || (v < i && v >= n_lo)) continue;
          int lo = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1)
            if (sh_cols[w][lo + step - 1] < v) lo += step;
          tslot[t] = lo;
          tk[t] = K;
          ++t;
          if (!kFill) atomicAdd(&sh_cnt[w][lo], 1);
        }
      }
      if (kFill) {
        for (int sl = 0; sl < ds; ++sl) {  // warp-uniform: lane order = ascending face order
          int K = -1;
#pragma unroll
          for (int t = 0; t < 4; ++t) K = (tslot[t] == sl) ? tk[t] : K;
          const unsigned m = __ballot_sync(0xffffffffu, K >= 0);
          if (K >= 0) prog[sh_cnt[w][sl] + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(k | (K << 13));
          __syncwarp();
          if (lane == 0) sh_cnt[w][sl] += __popc(m);
          __syncwarp();
        }
      }
    }
    __syncwarp();
    if (!kFill && lane < ds) cnt[P + lane] = sh_cnt[w][lane];
    __syncwarp();
  }
}

// Fast path, warp per own node i with <= 32 stored blocks (diagonal + j > i + halo j < n_lo),
// driven by the assembly program.  Rounds of 32 records (faces of F(i), or tets for FEM-T4;
// ascending):
//   load: the warp copies the round's 32 records (128 B each) into shared memory with coalesced
//      16-byte cp.async (8 warp instructions);
//   diagonal: lane = face, s_i s_i^T into the lane's partial sum (fixed warp tree at the end);
//   off-diagonal: lane = stored slot walks its program entries of the round (ascending face),
//      adding s_i s_K^T; rows with <= 16 stored blocks give every slot two lanes, one for the
//      even and one for the odd entries, combined at the end in that order.
// Summation order is fixed by the program: results do not depend on timing.
constexpr int kRowWarps = 4;
#ifndef FSFEM_ASM_MINB
#define FSFEM_ASM_MINB 8
#endif
// Shared-memory record stride (doubles).  128-B records at a 128-B stride put every record's
// s_K in the same banks (32-way conflicts when the lanes of a warp read the same K of different
// records).  18 doubles (144 B) spreads them over 8 bank offsets with 16-B copies: 581 us vs
// 806 us at 16 and 654 us at 17 (odd stride: conflict-free reads but 8-B copies), cfg4.
#ifndef FSFEM_ASM_STRIDE
#define FSFEM_ASM_STRIDE 18
#endif
constexpr int kSh = FSFEM_ASM_STRIDE;

__global__ void __launch_bounds__(kRowWarps * 32, FSFEM_ASM_MINB) k_assemble_rows3(
    const int64_t* __restrict__ sptr, const int32_t* __restrict__ snbr, const int64_t* __restrict__ nf_ptr,
    const int32_t* __restrict__ nf_idx, const uint8_t* __restrict__ nf_pi, const int32_t* __restrict__ blk_ent,
    const uint16_t* __restrict__ prog, const double* __restrict__ face_s, int64_t n_lo, int64_t nloc, double lam,
    double mu, double* __restrict__ vals) {
  __shared__ __align__(16) double sh_rec[kRowWarps][32][kSh];
  __shared__ uint8_t sh_pi[kRowWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t il = blockIdx.x * (int64_t)kRowWarps + w; il < nloc; il += (int64_t)gridDim.x * kRowWarps) {
    const int32_t self = static_cast<int32_t>(n_lo + il);
    const int64_t P = sptr[il];
    const int ds = static_cast<int>(sptr[il + 1] - P);
    if (ds > 32) continue;  // generic path
    const bool split = ds <= 16;
    const int slot = split ? (lane & 15) : lane;
    const int step = split ? 2 : 1;
    int e = 0, e_end = 0;
    if (slot < ds) {
      e = blk_ent[P + slot] + (split ? (lane >> 4) : 0);
      e_end = blk_ent[P + slot + 1];
    }
    uint32_t ent = e < e_end ? prog[e] : 0xffffu;
    const int32_t my_col = lane < ds ? snbr[P + lane] : -1;
    const int64_t f0 = nf_ptr[il];
    const int nfc = static_cast<int>(nf_ptr[il + 1] - f0);
    double d[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // diagonal partial: xx yy zz xy xz yz
    double M[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) M[q] = 0.0;
    for (int rb = 0; rb < nfc; rb += 32) {
      const int nact = min(32, nfc - rb);
      const int32_t myr = lane < nact ? nf_idx[f0 + rb + lane] : 0;
      const int mypi = lane < nact ? nf_pi[f0 + rb + lane] : 0;
      if (kSh % 2 == 0) {  // 16-B pieces (record slots 16-B aligned)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int c = lane + 32 * q;
          const int k = c >> 3, part = c & 7;
          const int32_t r = __shfl_sync(0xffffffffu, myr, k);
          if (k < nact) {
            const double2* src = reinterpret_cast<const double2*>(face_s + kRec * static_cast<int64_t>(r)) + part;
            const uint32_t dst =
                static_cast<uint32_t>(__cvta_generic_to_shared(&sh_rec[w][k][0])) + 16u * static_cast<uint32_t>(part);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          }
        }
      } else {  // 8-B pieces (odd stride)
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int c = lane + 32 * q;
          const int k = c >> 4, part = c & 15;
          const int32_t r = __shfl_sync(0xffffffffu, myr, k);
          if (k < nact) {
            const double* src = face_s + kRec * static_cast<int64_t>(r) + part;
            const uint32_t dst =
                static_cast<uint32_t>(__cvta_generic_to_shared(&sh_rec[w][k][0])) + 8u * static_cast<uint32_t>(part);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
          }
        }
      }
      sh_pi[w][lane] = static_cast<uint8_t>(mypi);
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      if (lane < nact) {
        const double* sf = sh_rec[w][lane];
        const double s0 = sf[3 * mypi], s1 = sf[3 * mypi + 1], s2 = sf[3 * mypi + 2];
        d[0] = fma(s0, s0, d[0]);
        d[1] = fma(s1, s1, d[1]);
        d[2] = fma(s2, s2, d[2]);
        d[3] = fma(s0, s1, d[3]);
        d[4] = fma(s0, s2, d[4]);
        d[5] = fma(s1, s2, d[5]);
      }
      const uint32_t kend = static_cast<uint32_t>(rb + 32);
      while ((ent & 0x1fffu) < kend) {  // (0xffff: no more entries; its k = 8191 >= any kend)
        const int kl = static_cast<int>(ent & 0x1fffu) - rb, K = static_cast<int>(ent >> 13);
        e += step;
        const uint32_t nxt = e < e_end ? prog[e] : 0xffffu;
        const double* rf = sh_rec[w][kl];
        const int pb = sh_pi[w][kl];
        const double a0 = rf[3 * pb], a1 = rf[3 * pb + 1], a2 = rf[3 * pb + 2];
        const double c0 = rf[3 * K], c1 = rf[3 * K + 1], c2 = rf[3 * K + 2];
        M[0] = fma(a0, c0, M[0]);
        M[1] = fma(a0, c1, M[1]);
        M[2] = fma(a0, c2, M[2]);
        M[3] = fma(a1, c0, M[3]);
        M[4] = fma(a1, c1, M[4]);
        M[5] = fma(a1, c2, M[5]);
        M[6] = fma(a2, c0, M[6]);
        M[7] = fma(a2, c1, M[7]);
        M[8] = fma(a2, c2, M[8]);
        ent = nxt;
      }
      __syncwarp();
    }
    if (split) {  // slot s = (even entries) + (odd entries): lane s adds lane s+16's partial
#pragma unroll
      for (int q = 0; q < 9; ++q) M[q] += __shfl_down_sync(0xffffffffu, M[q], 16);
    }
    // diagonal block: fixed warp tree of the per-lane partial sums
#pragma unroll
    for (int q = 0; q < 6; ++q) d[q] = warp_sum(d[q]);
    double* blocks = vals + 9 * P;
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

// Assembly program of the pattern (once; pattern.cuh).  rec_a/rec_b: FS face_nodes/face_opp,
// FEM-T4 tets/unused.  Returns the error word (kNoError if fine).
void build_assembly_program(Pattern& pat, const int32_t* rec_a, const int32_t* rec_b, bool tet,
                            DevBuf<unsigned char>& scratch, unsigned long long* h_flags, cudaStream_t s) {
  const int64_t nloc = pat.nloc, nsb = pat.nsb;
  pat.nf_pi.ensure(std::max<int64_t>(pat.nfi, 1));
  pat.blk_ent.ensure(nsb + 1);
  const size_t tb = scan_tmp_bytes(nsb + 1);
  const size_t o_cnt = 0, o_flags = (sizeof(int32_t) * (nsb + 1) + 255) & ~size_t(255),
               o_tmp = o_flags + 256;
  unsigned char* base = scratch.ensure(o_tmp + tb);
  int32_t* cnt = reinterpret_cast<int32_t*>(base + o_cnt);
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(base + o_flags);
  FS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nsb + 1), s));
  FS_CUDA(cudaMemsetAsync(flags, 0xff, sizeof(unsigned long long), s));
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, kProgWarps), 32LL * num_sms())));
  if (nloc > 0) {
    k_prog<false><<<g, kProgWarps * 32, 0, s>>>(pat.sptr.get(), pat.snbr.get(), pat.nf_ptr.get(), pat.nf_idx.get(), rec_a, rec_b,
                                    tet, pat.n_lo, nloc, pat.nf_pi.get(), cnt, nullptr, nullptr, flags);
    FS_LAUNCH_CHECK();
  }
  exclusive_scan_i32(cnt, pat.blk_ent.get(), nsb, s, base + o_tmp, tb);
  int32_t total = 0;
  FS_CUDA(cudaMemcpyAsync(&total, pat.blk_ent.get() + nsb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaMemcpyAsync(h_flags, flags, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  if (h_flags[0] != kNoError) return;
  pat.prog.ensure(std::max<int64_t>(total, 1));
  if (nloc > 0) {
    k_prog<true><<<g, kProgWarps * 32, 0, s>>>(pat.sptr.get(), pat.snbr.get(), pat.nf_ptr.get(), pat.nf_idx.get(), rec_a, rec_b,
                                   tet, pat.n_lo, nloc, nullptr, nullptr, pat.blk_ent.get(), pat.prog.get(), flags);
    FS_LAUNCH_CHECK();
  }
  pat.have_prog = true;
}

// rec_a/rec_b: FS (kTet = false) face_nodes/face_opp; FEM-T4 (tet = true) tets/unused.
void assemble_rows_device(const Pattern& pat, const int32_t* face_nodes, const int32_t* face_opp,
                          const double* face_s, double lam, double mu, double* vals, bool tet, cudaStream_t s) {
  const int64_t nloc = pat.nloc;
  if (nloc == 0) return;
  // Persistent grid of exactly the resident CTAs: warp w takes nodes w, w + W, ... so the nodes in
  // flight form one contiguous window that slides forward; the field nodes of a face (which span
  // less than two windows in a banded numbering) are then assembled close together in time and
  // the face's record is re-read from L2, not DRAM.
  static int per_sm = 0;
  if (per_sm == 0) FS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_assemble_rows3, kRowWarps * 32, 0));
  const int g2 = static_cast<int>(
      std::min<int64_t>(ceil_div(nloc, kRowWarps), static_cast<int64_t>(std::max(1, per_sm)) * num_sms()));
  k_assemble_rows3<<<std::max(g2, 1), kRowWarps * 32, 0, s>>>(pat.sptr.get(), pat.snbr.get(), pat.nf_ptr.get(),
                                                              pat.nf_idx.get(), pat.nf_pi.get(), pat.blk_ent.get(),
                                                              pat.prog.get(), face_s, pat.n_lo, nloc, lam, mu, vals);
  FS_LAUNCH_CHECK();
  if (pat.max_row_blocks > 32) {
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nloc * 32, 256), 32LL * num_sms()));
    auto k1 = tet ? k_assemble_rows<true> : k_assemble_rows<false>;
    k1<<<std::max(grid, 1), 256, 0, s>>>(pat.sptr.get(), pat.snbr.get(), pat.nf_ptr.get(), pat.nf_idx.get(),
                                         face_nodes, face_opp, face_s, pat.n_lo, nloc, lam, mu, vals, 32);
    FS_LAUNCH_CHECK();
  }
}

void tet_s_device(const double* xyz, const int32_t* tets, int64_t nt, double* tet_s, double* tet_V, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nt, 256), 16LL * num_sms()));
  k_tet_s<<<std::max(grid, 1), 256, 0, s>>>(xyz, tets, nt, tet_s, tet_V);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
