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

// =============================================================================================
// Tile assembly (S2-S4 + S6 in one kernel; DESIGN.md §6 "assembly").
//
// The own nodes are ordered along a Morton curve of their coordinates and cut into tiles of
// <= kTileRows rows.  The union U of the tile rows' domain lists F(i) (faces -- tets for FEM-T4 --
// whose field holds a tile row) is the only geometry a tile needs: the kernel computes
// s_K = (V b_K)/sqrt(V) of every domain of U ONCE into shared memory from the coordinates of the
// tile's vertices (staged in shared memory too), then sums every stored block of the tile rows
// from shared memory and writes the rows' values.  No per-domain record goes to HBM.
//
// Warp specialisation, one CTA per SM, two tile buffers: producer warps stage tile j+1 (blob,
// vertex coordinates, s records) while consumer warps sum and write tile j.
//
// Summation order (reading Q26) -- a function of the block alone, not of the tile, the rank's
// range or the row length, so results are bitwise reproducible AND partition-invariant:
//   off-diagonal block (i, j): the domains of F(i) n F(j) in ascending id, in sequence;
//   diagonal block (i, i): the domains of F(i) in ascending id split into kDiagSplit strided
//     sub-lists (entries q, q + kDiagSplit, ...), each summed in sequence, then the sub-list sums
//     added in q order.
// Each block is then K_ij = lam M + mu M^T + mu tr(M) I (M-form, reading Q25).
//
// Per-tile blob (built once per pattern by k_tile_build, read once per assembly):
//   TileHdr | rows [nrows] (P = first stored block of the row, il) | verts int32 [nverts] (tile
//   rows first) | fv u8 [ndom][5] (local vertex of field position p, 255 = none) |
//   tasks [ntask] (entry start, slot, count, row, sub-list) | ent u16 [nent] ((local domain << 5)
//   | 5 pos_i + pos_j), the entries of every stored block (rows in tile order, slots in order).
// Local domain order = ascending domain id.  Tasks are stored longest first (load balance; which
// thread runs a task does not change its sum).
// =============================================================================================
#ifndef FSFEM_ASM_SPLIT
#define FSFEM_ASM_SPLIT 1
#endif
constexpr int kTileRows = 16;
constexpr int kMaxDom = 640;      // domains per tile (shared-memory s records: 120 B each)
constexpr int kMaxVerts = 254;    // u8 local vertex ids, 255 = none
constexpr int kDiagCap = 2048;    // sum over the tile rows of |F(i)|
constexpr int kMaxBlk = 767;      // stored blocks of the tile rows
constexpr int kMaxTask = 1024;
#ifndef FSFEM_DIAG_SPLIT
#define FSFEM_DIAG_SPLIT 4
#endif
constexpr int kDiagSplit = FSFEM_DIAG_SPLIT;  // strided sub-lists of a diagonal block
constexpr int kBlobCap = 14336;   // bytes of one tile blob
constexpr int kAsmWarps = 16;     // 8 producer + 8 consumer warps
constexpr int kAsmThreads = 32 * kAsmWarps;
constexpr int kGroup = kAsmThreads / 2;

struct TileHdr {
  int32_t nrows, nverts, ndom, ntask, nent, pad0, pad1, pad2;
};
struct TileRow {
  int64_t P;  // first stored block of the row (index into vals / 9)
  int32_t il;
  int32_t sdiag;  // slot of the diagonal block, -1 for a row without blocks (a node in no tet)
};
struct TileTask {
  uint16_t estart, slot;
  uint8_t count, row, sub, pad;  // sub = 255: off-diagonal block (stride 1); else diagonal sub-list
};
__host__ __device__ __forceinline__ constexpr int al16(int x) { return (x + 15) & ~15; }
struct TileLayout {
  int o_rows, o_verts, o_fv, o_task, o_ent, bytes;
  __host__ __device__ TileLayout(int nrows, int nverts, int ndom, int ntask, int nent) {
    o_rows = 32;
    o_verts = al16(o_rows + 16 * nrows);
    o_fv = al16(o_verts + 4 * nverts);
    o_task = al16(o_fv + 5 * ndom);
    o_ent = al16(o_task + 8 * ntask);
    bytes = al16(o_ent + 2 * nent);
  }
};

// ---- builder (once per pattern) ---------------------------------------------------------------
constexpr int kBldThreads = 256;
constexpr int kHashD = 2048;  // domain hash slots (>= 2 x the tile's list entries cap kDiagCap / 1)
constexpr int kHashV = 1024;  // vertex hash slots (>= 4 x kMaxVerts)

__device__ __forceinline__ unsigned hslot(int32_t x, unsigned mask) {
  return (static_cast<unsigned>(x) * 2654435761u >> 7) & mask;
}
// Insert x into the open-addressing set keys[0..mask] (empty = -1); duplicates collapse.
// Returns true if x was new.
__device__ __forceinline__ bool hinsert(int32_t* keys, unsigned mask, int32_t x) {
  unsigned h = hslot(x, mask);
  for (;;) {
    const int32_t old = atomicCAS(&keys[h], -1, x);
    if (old == -1) return true;
    if (old == x) return false;
    h = (h + 1) & mask;
  }
}
__device__ __forceinline__ int hfind(const int32_t* keys, const int32_t* idx, unsigned mask, int32_t x) {
  unsigned h = hslot(x, mask);
  while (keys[h] != x) h = (h + 1) & mask;
  return idx[h];
}

// Exclusive CTA scan of one int per thread (kBldThreads threads); *total = sum.
__device__ int cta_excl_scan(int v, int* total) {
  __shared__ int ws[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  int base = 0, tot = 0;
  for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) {
    if (k < w) base += ws[k];
    tot += ws[k];
  }
  __syncthreads();
  *total = tot;
  return base + inc - v;
}

// Slot of x in the open-addressing set keys[0..mask] (inserted if absent).
__device__ __forceinline__ int hinsert_at(int32_t* keys, unsigned mask, int32_t x) {
  unsigned h = hslot(x, mask);
  for (;;) {
    const int32_t old = atomicCAS(&keys[h], -1, x);
    if (old == -1 || old == x) return static_cast<int>(h);
    h = (h + 1) & mask;
  }
}
// idx of x, or -1 if x is not in the set (an empty slot ends the probe: no deletions).
__device__ __forceinline__ int hfind_or(const int32_t* keys, const int32_t* idx, unsigned mask, int32_t x) {
  unsigned h = hslot(x, mask);
  for (unsigned n = 0; n <= mask; ++n) {
    const int32_t k = keys[h];
    if (k == x) return idx[h];
    if (k == -1) return -1;
    h = (h + 1) & mask;
  }
  return -1;
}

// Shared memory of the builder (int32 words unless noted).
constexpr int kStStride = 256;  // slot table row stride (local vertex ids < kMaxVerts < 256)
constexpr int kBldSmem = static_cast<int>(sizeof(int32_t)) *
                             (2 * kHashD + kMaxDom + 2 * kHashV + kMaxVerts + kTileRows + 2 * (kMaxBlk + 1) +
                              2 * kMaxTask) +
                         al16(5 * kMaxDom) + 2 * kTileRows * kStStride;

// One CTA per tile, one pass: the blob at blob + t * kBlobCap and its size into size[t] (or
// -1 = too big for the caps: split the tile, -2 = a single row that cannot fit: UNSUPPORTED).
// The tile's domains and vertices are collected in shared-memory hash sets: their local numbering
// is arbitrary (it only names shared-memory slots), while every summation order is fixed by the
// rows' ascending domain lists F(i).  The tile rows enter the vertex set first with local ids
// 0..nrows-1; the slot of stored column J in row r comes from a table indexed by J's local id
// (filled from the rows' stored column lists), not from a search of the global list.
__global__ void __launch_bounds__(kBldThreads) k_tile_build(
    const int32_t* __restrict__ order, const int2* __restrict__ trange, const int32_t* __restrict__ which,
    int64_t nwork, const int64_t* __restrict__ nf_ptr, const int32_t* __restrict__ nf_idx, const int32_t* __restrict__ rec_a,
    const int32_t* __restrict__ rec_b, bool tet, const int64_t* __restrict__ sptr, const int32_t* __restrict__ snbr,
    const int32_t* __restrict__ sdiag, int64_t n_lo, int64_t* __restrict__ size, unsigned char* __restrict__ blob) {
  extern __shared__ __align__(16) unsigned char bsm[];
  int32_t* HK = reinterpret_cast<int32_t*>(bsm);  // [kHashD] domain keys
  int32_t* HI = HK + kHashD;                       // [kHashD] local domain index
  int32_t* U = HI + kHashD;                        // [kMaxDom] local -> domain id
  int32_t* VK = U + kMaxDom;                       // [kHashV] vertex keys
  int32_t* VI = VK + kHashV;                       // [kHashV] local vertex index (-1: not numbered yet)
  int32_t* VL = VI + kHashV;                       // [kMaxVerts + kTileRows] local -> node id
  int32_t* bcnt = VL + kMaxVerts + kTileRows;      // [kMaxBlk + 1] entries per block
  int32_t* cur = bcnt + kMaxBlk + 1;               // [kMaxBlk + 1] entry offsets / cursors
  int32_t* tkey = cur + kMaxBlk + 1;               // [kMaxTask] task keys (count, index)
  int32_t* tinfo = tkey + kMaxTask;                // [kMaxTask] row << 24 | sub-list << 16 | slot
  unsigned char* FV = reinterpret_cast<unsigned char*>(tinfo + kMaxTask);      // [kMaxDom][5] local vertices
  uint16_t* ST = reinterpret_cast<uint16_t*>(FV + al16(5 * kMaxDom));          // [kTileRows][kStStride] slots
  __shared__ int32_t rnode[kTileRows], ril[kTileRows], rds[kTileRows], rsd[kTileRows], rbb[kTileRows + 1];
  __shared__ int64_t rP[kTileRows], rF[kTileRows + 1];
  __shared__ int sh_flag, sh_ntask, sh_nent, sh_nv;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
    const int64_t t = which ? which[wi] : wi;  // tile t = own rows order[trange[t].x, trange[t].y)
    const int2 trg = trange[t];
    const int nrows = trg.y - trg.x;
    if (w == 0) {  // rows: lane r loads row r, lane scans give the block / domain-list offsets
      int ds = 0;
      int64_t nfr = 0;
      if (lane < nrows) {
        const int32_t il = order[trg.x + lane];
        const int64_t P = sptr[il];
        ds = static_cast<int>(sptr[il + 1] - P);
        nfr = nf_ptr[il + 1] - nf_ptr[il];
        ril[lane] = il;
        rnode[lane] = static_cast<int32_t>(n_lo + il);
        rP[lane] = P;
        rds[lane] = ds;
        rsd[lane] = ds > 0 ? sdiag[il] : -1;
      }
      int bb = ds;
      int64_t fs = nfr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, bb, o);
        const int64_t z = __shfl_up_sync(0xffffffffu, fs, o);
        if (lane >= o) {
          bb += y;
          fs += z;
        }
      }
      if (lane < nrows) {
        rbb[lane] = bb - ds;
        rF[lane] = fs - nfr;
      }
      if (lane == 31) {
        rbb[nrows] = bb;
        rF[nrows] = fs;
        sh_flag = (fs > kDiagCap || bb > kMaxBlk) ? 1 : 0;
        sh_nv = nrows;
      }
    }
    for (int k = threadIdx.x; k < kHashD; k += blockDim.x) HK[k] = -1;
    for (int k = threadIdx.x; k < kHashV; k += blockDim.x) {
      VK[k] = -1;
      VI[k] = -1;
    }
    __syncthreads();
    if (sh_flag) {
      if (threadIdx.x == 0) size[t] = -(nrows > 1 ? 1 : 2);
      __syncthreads();
      continue;
    }
    // domains: hash set of the rows' lists; the rows enter the vertex set with local ids 0..nrows-1
    const int nA = static_cast<int>(rF[nrows]);
    for (int k = threadIdx.x; k < nA; k += blockDim.x) {
      int r = 0;
      while (rF[r + 1] <= k) ++r;
      hinsert(HK, kHashD - 1, nf_idx[nf_ptr[ril[r]] + (k - rF[r])]);
    }
    if (threadIdx.x < nrows) VI[hinsert_at(VK, kHashV - 1, rnode[threadIdx.x])] = threadIdx.x;
    __syncthreads();
    int ndom = 0;
    {
      constexpr int per = kHashD / kBldThreads;
      int c = 0;
      for (int q = 0; q < per; ++q) c += HK[threadIdx.x * per + q] >= 0 ? 1 : 0;
      int base = cta_excl_scan(c, &ndom);
      for (int q = 0; q < per; ++q) {
        const int h = threadIdx.x * per + q;
        if (HK[h] >= 0) {
          HI[h] = base;
          if (base < kMaxDom) U[base] = HK[h];
          ++base;
        }
      }
    }
    __syncthreads();
    if (ndom > kMaxDom) {
      if (threadIdx.x == 0) size[t] = -(nrows > 1 ? 1 : 2);
      __syncthreads();
      continue;
    }
    for (int k = threadIdx.x; k < ndom; k += blockDim.x) {
      int32_t fld[5];
      field_of(rec_a, rec_b, tet, U[k], fld);
#pragma unroll
      for (int p = 0; p < 5; ++p)  // the set stays at most half full (a tile with more is split)
        if (fld[p] >= 0 && sh_nv < kHashV / 2 && hinsert(VK, kHashV - 1, fld[p])) atomicAdd(&sh_nv, 1);
    }
    __syncthreads();
    if (sh_nv >= kHashV / 2) {
      if (threadIdx.x == 0) size[t] = -(nrows > 1 ? 1 : 2);
      __syncthreads();
      continue;
    }
    // vertices: tile rows first (local r, already numbered), the others after them
    int nverts = 0;
    {
      constexpr int per = kHashV / kBldThreads;
      int c = 0;
      for (int q = 0; q < per; ++q) {
        const int h = threadIdx.x * per + q;
        c += (VK[h] >= 0 && VI[h] < 0) ? 1 : 0;
      }
      int no = 0;
      int base = nrows + cta_excl_scan(c, &no);
      for (int q = 0; q < per; ++q) {
        const int h = threadIdx.x * per + q;
        if (VK[h] >= 0 && VI[h] < 0) {
          VI[h] = base;
          if (base < kMaxVerts + kTileRows) VL[base] = VK[h];
          ++base;
        }
      }
      for (int r = threadIdx.x; r < nrows; r += blockDim.x) VL[r] = rnode[r];
      nverts = nrows + no;
    }
    __syncthreads();
    if (nverts > kMaxVerts) {
      if (threadIdx.x == 0) size[t] = -(nrows > 1 ? 1 : 2);
      __syncthreads();
      continue;
    }
    // local vertices of every domain's field positions; slot table of the rows' stored columns
    for (int k = threadIdx.x; k < ndom; k += blockDim.x) {
      int32_t fld[5];
      field_of(rec_a, rec_b, tet, U[k], fld);
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        const int v = fld[p] >= 0 ? hfind_or(VK, VI, kHashV - 1, fld[p]) : -1;
        FV[5 * k + p] = static_cast<unsigned char>(v >= 0 ? v : 255);
      }
    }
    for (int r = w; r < nrows; r += kBldThreads / 32) {
      const int64_t P = rP[r];
      for (int s = lane; s < rds[r]; s += 32) {
        const int v = hfind_or(VK, VI, kHashV - 1, snbr[P + s]);
        if (v >= 0) ST[r * kStStride + v] = static_cast<uint16_t>(s);
      }
    }
    for (int b = threadIdx.x; b <= kMaxBlk; b += blockDim.x) bcnt[b] = 0;
    __syncthreads();
    // entries per stored block: off-diagonal (i, J): one per domain of F(i) holding J (stored J);
    // diagonal: one per domain of F(i).  Warp per row, lane per domain.
    for (int r = w; r < nrows; r += kBldThreads / 32) {
      const int32_t i = rnode[r];
      const int64_t fb = nf_ptr[ril[r]];
      const int len = static_cast<int>(rF[r + 1] - rF[r]);
      for (int k0 = 0; k0 < len; k0 += 32) {
        const int k = k0 + lane;
        if (k < len) {
          const int kl = hfind(HK, HI, kHashD - 1, nf_idx[fb + k]);
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            const int v = FV[5 * kl + q];
            if (v == 255) continue;
            const int32_t J = VL[v];
            if (J < i && J >= n_lo) continue;
            const int slot = v == r ? rsd[r] : ST[r * kStStride + v];
            atomicAdd(&bcnt[rbb[r] + slot], 1);
          }
        }
      }
    }
    __syncthreads();
    {  // entry offsets and tasks (longest first; ties in block order): CTA scans over the blocks
      const int nblk = rbb[nrows];
      constexpr int per = (kMaxBlk + 1) / kBldThreads;  // 3 blocks per thread
      int ce = 0, ct = 0;
      bool ok = true;
      int rr[per], ss[per];
      for (int q = 0; q < per; ++q) {
        const int b = threadIdx.x * per + q;
        rr[q] = -1;
        ss[q] = 0;
        if (b < nblk) {
          int r = 0;
          while (rbb[r + 1] <= b) ++r;
          rr[q] = r;
          ss[q] = b - rbb[r];
          ce += bcnt[b];
          const bool dg = ss[q] == rsd[r];
          ct += dg ? kDiagSplit : 1;
          ok = ok && bcnt[b] <= (dg ? 255 * kDiagSplit : 255);
        }
      }
      int tot_e = 0, tot_t = 0;
      int e0 = cta_excl_scan(ce, &tot_e);
      int t0 = cta_excl_scan(ct, &tot_t);
      ok = __syncthreads_and(ok) && tot_t <= kMaxTask && tot_e < 65536;
      for (int q = 0; q < per; ++q) {
        const int b = threadIdx.x * per + q;
        if (rr[q] < 0) continue;
        cur[b] = e0;
        e0 += bcnt[b];
        if (!ok) continue;
        if (ss[q] == rsd[rr[q]]) {
          for (int qq = 0; qq < kDiagSplit; ++qq) {
            const int c = (bcnt[b] - qq + kDiagSplit - 1) / kDiagSplit;
            tkey[t0] = ((1023 - c) << 20) | t0;
            tinfo[t0] = (rr[q] << 24) | (qq << 16) | ss[q];
            ++t0;
          }
        } else {
          tkey[t0] = ((1023 - bcnt[b]) << 20) | t0;
          tinfo[t0] = (rr[q] << 24) | (255 << 16) | ss[q];
          ++t0;
        }
      }
      if (threadIdx.x == 0) {
        sh_nent = tot_e;
        sh_ntask = tot_t;
        sh_flag = ok ? 0 : 1;
      }
    }
    __syncthreads();
    const int nent = sh_nent, ntask = sh_ntask;
    const TileLayout L(nrows, nverts, ndom, ntask, nent);
    const bool ok = !sh_flag && nverts <= kMaxVerts && L.bytes <= kBlobCap;
    if (threadIdx.x == 0) size[t] = ok ? L.bytes : -(nrows > 1 ? 1 : 2);
    if (!ok) {
      __syncthreads();
      continue;
    }
    unsigned char* bl = blob + t * static_cast<int64_t>(kBlobCap);
    if (threadIdx.x == 0) {
      TileHdr h{nrows, nverts, ndom, ntask, nent, 0, 0, 0};
      *reinterpret_cast<TileHdr*>(bl) = h;
    }
    for (int r = threadIdx.x; r < nrows; r += blockDim.x)
      reinterpret_cast<TileRow*>(bl + L.o_rows)[r] = TileRow{rP[r], ril[r], rsd[r]};
    for (int v = threadIdx.x; v < nverts; v += blockDim.x) reinterpret_cast<int32_t*>(bl + L.o_verts)[v] = VL[v];
    for (int k = threadIdx.x; k < 5 * ndom; k += blockDim.x) bl[L.o_fv + k] = FV[k];
    {
      TileTask* tasks = reinterpret_cast<TileTask*>(bl + L.o_task);
      // rank of task a = #{keys < key_a}, key = (1023 - count) << 20 | a: a counting sort over the
      // 1024 count bins, then in-bin order by a (one warp, __match_any per round of 32 tasks).
      // The vertex hash set is dead here (FV and ST hold what is needed): its arrays are reused.
      int32_t* hist = VK;  // [1024] bin sizes -> bin starts
      int32_t* run = VI;   // [1024] tasks of each bin ranked so far
      for (int b = threadIdx.x; b < 1024; b += blockDim.x) {
        hist[b] = 0;
        run[b] = 0;
      }
      __syncthreads();
      for (int a = threadIdx.x; a < ntask; a += blockDim.x) atomicAdd(&hist[tkey[a] >> 20], 1);
      __syncthreads();
      {
        static_assert(kBldThreads * 4 == 1024, "four bins per thread");
        int v[4], sum = 0, tot = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[q] = hist[4 * threadIdx.x + q];
          sum += v[q];
        }
        int base = cta_excl_scan(sum, &tot);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hist[4 * threadIdx.x + q] = base;
          base += v[q];
        }
      }
      __syncthreads();
      if (w == 0) {
        for (int a0 = 0; a0 < ntask; a0 += 32) {
          const int a = a0 + lane;
          const int bin = a < ntask ? (tkey[a] >> 20) : 1024 + lane;  // padding lanes match nobody
          const unsigned peers = __match_any_sync(0xffffffffu, bin);
          const int before = __popc(peers & ((1u << lane) - 1u));
          if (a < ntask) tkey[a] = hist[bin] + run[bin] + before;  // the key becomes the rank
          __syncwarp();
          if (a < ntask && lane == 31 - __clz(peers)) run[bin] += __popc(peers);
          __syncwarp();
        }
      }
      __syncthreads();
      for (int a = threadIdx.x; a < ntask; a += blockDim.x) {
        const int rank = tkey[a];
        const int r = tinfo[a] >> 24, q = (tinfo[a] >> 16) & 255, sl = tinfo[a] & 0xffff;
        const int b = rbb[r] + sl;
        TileTask tk;
        tk.slot = static_cast<uint16_t>(sl);
        tk.row = static_cast<uint8_t>(r);
        tk.sub = static_cast<uint8_t>(q);
        tk.pad = 0;
        if (q == 255) {
          tk.estart = static_cast<uint16_t>(cur[b]);
          tk.count = static_cast<uint8_t>(bcnt[b]);
        } else {
          tk.estart = static_cast<uint16_t>(cur[b] + q);
          tk.count = static_cast<uint8_t>((bcnt[b] - q + kDiagSplit - 1) / kDiagSplit);
        }
        tasks[rank] = tk;
      }
    }
    __syncthreads();
    // entries: per row, rounds of 32 domains in ascending id; slot by slot, the lanes holding the
    // slot write in lane (= ascending domain) order
    uint16_t* ent = reinterpret_cast<uint16_t*>(bl + L.o_ent);
    for (int r = w; r < nrows; r += kBldThreads / 32) {
      const int32_t i = rnode[r];
      const int64_t fb = nf_ptr[ril[r]];
      const int len = static_cast<int>(rF[r + 1] - rF[r]);
      const int ds = rds[r];
      for (int k0 = 0; k0 < len; k0 += 32) {
        const int k = k0 + lane;
        int tslot[5] = {-1, -1, -1, -1, -1}, tcode[5] = {0, 0, 0, 0, 0}, kl = 0;
        if (k < len) {
          kl = hfind(HK, HI, kHashD - 1, nf_idx[fb + k]);
          int pi = 0;
#pragma unroll
          for (int p = 0; p < 5; ++p) pi = FV[5 * kl + p] == r ? p : pi;
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            const int v = FV[5 * kl + q];
            if (v == 255) continue;
            const int32_t J = VL[v];
            if (J < i && J >= n_lo) continue;
            tslot[q] = v == r ? rsd[r] : ST[r * kStStride + v];
            tcode[q] = 5 * pi + q;
          }
        }
        // slots touched by this round, lowest first (warp-uniform loop over the union)
        unsigned long long lo_mask = 0ull;  // slots < 64 as a bit set; others via the slow loop
        bool big = false;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          if (tslot[q] >= 64) big = true;
          else if (tslot[q] >= 0) lo_mask |= 1ull << tslot[q];
        }
        unsigned long long all = lo_mask;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) all |= __shfl_xor_sync(0xffffffffu, all, o);
        const bool any_big = __any_sync(0xffffffffu, big);
        auto emit = [&](int sl) {
          int code = -1;
#pragma unroll
          for (int q = 0; q < 5; ++q) code = tslot[q] == sl ? tcode[q] : code;
          const unsigned m = __ballot_sync(0xffffffffu, code >= 0);
          const int b = rbb[r] + sl;
          if (code >= 0) ent[cur[b] + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>((kl << 5) | code);
          __syncwarp();
          if (lane == 0) cur[b] += __popc(m);
          __syncwarp();
        };
        while (all) {
          const int sl = __ffsll(static_cast<long long>(all)) - 1;
          all &= all - 1ull;
          emit(sl);
        }
        if (any_big)
          for (int sl = 64; sl < ds; ++sl) emit(sl);
      }
    }
    __syncthreads();
  }
}

// ---- numeric kernel ---------------------------------------------------------------------------
constexpr int kSRecBytes = kMaxDom * 15 * 8;
constexpr int kXBytes = al16(kMaxVerts * 3 * 8);
constexpr int kBlobSlots = 4;
constexpr int kAsmSmem = 2 * (kSRecBytes + kXBytes) + kBlobSlots * kBlobCap + kTileRows * kDiagSplit * 6 * 8 +
                         8 * kBlobSlots + 128;

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// M-form of one block (reading Q25): K = lam M + mu M^T + mu tr(M) I, M = sum s_i s_j^T.
__device__ __forceinline__ void mform_block(const double* M, double lam, double mu, double* out) {
  const double tr = M[0] + M[4] + M[8];
#pragma unroll
  for (int aa = 0; aa < 3; ++aa)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      double v = fma(lam, M[3 * aa + cc], mu * M[3 * cc + aa]);
      if (aa == cc) v = fma(mu, tr, v);
      out[3 * aa + cc] = v;
    }
}

// The same block written to global memory with 16-B stores (5 store instructions instead of 9;
// blocks are 72 B, so every other one starts 16-B aligned).
__device__ __forceinline__ void mform_block_store(const double* M, double lam, double mu, double* out) {
  double k[9];
  mform_block(M, lam, mu, k);
  if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    double2* o = reinterpret_cast<double2*>(out);
    o[0] = make_double2(k[0], k[1]);
    o[1] = make_double2(k[2], k[3]);
    o[2] = make_double2(k[4], k[5]);
    o[3] = make_double2(k[6], k[7]);
    out[8] = k[8];
  } else {
    out[0] = k[0];
    double2* o = reinterpret_cast<double2*>(out + 1);
    o[0] = make_double2(k[1], k[2]);
    o[1] = make_double2(k[3], k[4]);
    o[2] = make_double2(k[5], k[6]);
    o[3] = make_double2(k[7], k[8]);
  }
}

template <bool kTet>
__device__ __forceinline__ void domain_s(const double* __restrict__ X, const unsigned char* fv, double* out);

// K7 debug export: the dense stiffness of selected domains with the assembly's own
// arithmetic (domain_s, one M = s_I s_J^T per block, mform_block); thread per domain.
template <bool kTet>
__global__ void k_domain_stiffness(const double* __restrict__ xyz, const int32_t* __restrict__ rec_a,
                                   const int32_t* __restrict__ rec_b, const int64_t* __restrict__ ids, int64_t n,
                                   double lam, double mu, double* __restrict__ K, int32_t* __restrict__ field) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    int32_t fld[5];
    field_of(rec_a, rec_b, kTet, ids[q], fld);
    double X[15];
    unsigned char fv[5];
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      fv[p] = fld[p] >= 0 ? static_cast<unsigned char>(p) : 255;
      const int32_t v = fld[p] >= 0 ? fld[p] : fld[0];
      X[3 * p] = xyz[3 * (int64_t)v];
      X[3 * p + 1] = xyz[3 * (int64_t)v + 1];
      X[3 * p + 2] = xyz[3 * (int64_t)v + 2];
    }
    double sv[15];
    domain_s<kTet>(X, fv, sv);
    double* Kq = K + 225 * q;
    for (int I = 0; I < 5; ++I)
      for (int J = 0; J < 5; ++J) {
        double blk[9];
        if (fld[I] >= 0 && fld[J] >= 0) {
          double M[9];
#pragma unroll
          for (int aa = 0; aa < 3; ++aa)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) M[3 * aa + cc] = fma(sv[3 * I + aa], sv[3 * J + cc], 0.0);
          mform_block(M, lam, mu, blk);
        } else {
#pragma unroll
          for (int e = 0; e < 9; ++e) blk[e] = 0.0;
        }
#pragma unroll
        for (int aa = 0; aa < 3; ++aa)
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) Kq[15 * (3 * I + aa) + 3 * J + cc] = blk[3 * aa + cc];
      }
#pragma unroll
    for (int p = 0; p < 5; ++p) field[5 * q + p] = fld[p];
  }
}

// s_K of domain k from the staged coordinates.  FS: field (a, b, c, d, e) -- the face nodes and
// the vertices opposite the face in its tets (a, b, c, d) and (a, b, c, e); each tet's weights
// w_K = (V_e / 4) grad N_K^e = sign(det) (cross product of two edges) / 24 land on known field
// positions; s_K = (sum over the tets of w_K) / sqrt(V_f), V_f = sum |det| / 24 (closed form of
// Eq. 7, reading Q24).  FEM-T4: s_I = sqrt(V_e) grad N_I (reading Q25).
template <bool kTet>
__device__ __forceinline__ void domain_s(const double* __restrict__ X, const unsigned char* fv, double* out) {
  auto P = [&](int p, double& x, double& y, double& z) {
    const double* q = X + 3 * fv[p];
    x = q[0];
    y = q[1];
    z = q[2];
  };
  if (kTet) {
    double x0, y0, z0, x1, y1, z1, x2, y2, z2, x3, y3, z3;
    P(0, x0, y0, z0);
    P(1, x1, y1, z1);
    P(2, x2, y2, z2);
    P(3, x3, y3, z3);
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
    const double sc = sqrt(V) / det;
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      const double a = g[1][h] * sc, b = g[2][h] * sc, c = g[3][h] * sc;
      out[3 + h] = a;
      out[6 + h] = b;
      out[9 + h] = c;
      out[h] = -(a + b + c);
      out[12 + h] = 0.0;
    }
    return;
  }
  double ax, ay, az, bx, by, bz, cx, cy, cz, dx, dy, dz;
  P(0, ax, ay, az);
  P(1, bx, by, bz);
  P(2, cx, cy, cz);
  P(3, dx, dy, dz);
  const bool two = fv[4] != 255;
  double ex = 0.0, ey = 0.0, ez = 0.0;
  if (two) P(4, ex, ey, ez);
  const double e1x = bx - ax, e1y = by - ay, e1z = bz - az;
  const double e2x = cx - ax, e2y = cy - ay, e2z = cz - az;
  const double c3x = e1y * e2z - e1z * e2y, c3y = e1z * e2x - e1x * e2z, c3z = e1x * e2y - e1y * e2x;
  double g[5][3];
  double Vf;
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
  if (two) {  // tet (a, b, c, e)
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
#pragma unroll
  for (int K = 0; K < 5; ++K) {
    out[3 * K] = g[K][0] * rs;
    out[3 * K + 1] = g[K][1] * rs;
    out[3 * K + 2] = g[K][2] * rs;
  }
}

// Warps 0-7 produce tile j into S/X buffer j & 1 (s records from the coordinates; the blob of
// tile j + 2 is bulk-copied (TMA) into blob slot (j + 2) % 4 and the coordinates of tile j + 1
// gathered with cp.async meanwhile, so neither latency is on the producer's path), warps 8-15
// consume (tasks, writes).  Named barriers: 1 + b "buffer b full" (producers arrive, consumers
// sync), 3 + b "buffer b free" (consumers arrive, producers sync), 5 producers only, 6 consumers.
__device__ __forceinline__ uint32_t sm_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void tma_blob(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm_u32(dst)), "l"(src), "r"(bytes), "r"(sm_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   sm_u32(bar)), "r"(parity)
               : "memory");
}

template <bool kTet>
__global__ void __launch_bounds__(kAsmThreads, 1) k_asm_tile(const int64_t* __restrict__ tile_bytes,
                                                             const unsigned char* __restrict__ gblob, int64_t ntiles,
                                                             const double* __restrict__ xyz, double lam, double mu,
                                                             double* __restrict__ vals) {
  extern __shared__ __align__(128) unsigned char asm_sm[];
  double* Sb = reinterpret_cast<double*>(asm_sm);                                   // [2][kMaxDom * 15]
  double* Xb = reinterpret_cast<double*>(asm_sm + 2 * kSRecBytes);                  // [2][kXBytes / 8]
  unsigned char* Bb = asm_sm + 2 * kSRecBytes + 2 * kXBytes;                        // [kBlobSlots][kBlobCap]
  double* dpart = reinterpret_cast<double*>(Bb + kBlobSlots * kBlobCap);           // [rows][split][6]
  uint64_t* bars = reinterpret_cast<uint64_t*>(dpart + kTileRows * kDiagSplit * 6);  // [kBlobSlots]
  const int tid = threadIdx.x;
  const bool producer = tid < kGroup;
  const int gt = producer ? tid : tid - kGroup;  // thread index inside the group
  const int K = ntiles > blockIdx.x ? static_cast<int>((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto tile = [&](int j) { return blockIdx.x + static_cast<int64_t>(j) * gridDim.x; };
  auto blob_of = [&](int j) { return Bb + (j % kBlobSlots) * kBlobCap; };
  if (producer) {
    auto issue_blob = [&](int j) {  // one thread
      const int64_t t = tile(j);
      tma_blob(blob_of(j), gblob + t * static_cast<int64_t>(kBlobCap), static_cast<uint32_t>(tile_bytes[t]),
               &bars[j % kBlobSlots]);
    };
    auto wait_blob = [&](int j) { mbar_wait_parity(&bars[j % kBlobSlots], (j / kBlobSlots) & 1); };
    auto issue_x = [&](int j) {  // all producers: cp.async of the tile's vertex coordinates
      const unsigned char* blob = blob_of(j);
      const TileHdr h = *reinterpret_cast<const TileHdr*>(blob);
      const TileLayout L(h.nrows, h.nverts, h.ndom, h.ntask, h.nent);
      const int32_t* verts = reinterpret_cast<const int32_t*>(blob + L.o_verts);
      double* X = Xb + (j & 1) * (kXBytes / 8);
      for (int k = gt; k < 3 * h.nverts; k += kGroup) {
        const int v = k / 3, c = k - 3 * v;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sm_u32(X + k)),
                     "l"(xyz + 3 * static_cast<int64_t>(verts[v]) + c)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (gt == 0) {
      for (int k = 0; k < kBlobSlots; ++k)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(&bars[k])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (K > 0) issue_blob(0);
      if (K > 1) issue_blob(1);
    }
    named_sync(5, kGroup);
    if (K > 0) {
      wait_blob(0);
      issue_x(0);
    }
    for (int j = 0; j < K; ++j) {
      const int b = j & 1;
      if (j >= 2) named_sync(3 + b, kAsmThreads);  // consumers are done with tile j - 2
      if (gt == 0 && j + 2 < K) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_blob(j + 2);  // slot (j + 2) % 4 held tile j - 2
      }
      if (j + 1 < K) {
        wait_blob(j + 1);
        issue_x(j + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // tile j's coordinates landed
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      named_sync(5, kGroup);
      const unsigned char* blob = blob_of(j);
      const TileHdr h = *reinterpret_cast<const TileHdr*>(blob);
      const TileLayout L(h.nrows, h.nverts, h.ndom, h.ntask, h.nent);
      const unsigned char* fv = blob + L.o_fv;
      const double* X = Xb + b * (kXBytes / 8);
      double* S = Sb + b * (kSRecBytes / 8);
#ifndef FSFEM_ASM_SKIP
#define FSFEM_ASM_SKIP 0
#endif
      if (FSFEM_ASM_SKIP != 1) {
        // two domains per thread and pass (independent FP64 chains interleave)
        for (int k = gt; k < h.ndom; k += 2 * kGroup) {
          const int k2 = k + kGroup;
          double o1[15], o2[15];
          domain_s<kTet>(X, fv + 5 * k, o1);
          domain_s<kTet>(X, fv + 5 * min(k2, h.ndom - 1), o2);
#if FSFEM_ASM_SPLIT
          // split record layout: (x, y) of s_K as one 16-B pair at SA[5 k + K], z at SB[5 k + K]
          double2* SA = reinterpret_cast<double2*>(S);
          double* SB = S + 10 * kMaxDom;
#pragma unroll
          for (int K = 0; K < 5; ++K) {
            SA[5 * k + K] = make_double2(o1[3 * K], o1[3 * K + 1]);
            SB[5 * k + K] = o1[3 * K + 2];
          }
          if (k2 < h.ndom)
#pragma unroll
            for (int K = 0; K < 5; ++K) {
              SA[5 * k2 + K] = make_double2(o2[3 * K], o2[3 * K + 1]);
              SB[5 * k2 + K] = o2[3 * K + 2];
            }
#else
#pragma unroll
          for (int q = 0; q < 15; ++q) S[15 * k + q] = o1[q];
          if (k2 < h.ndom)
#pragma unroll
            for (int q = 0; q < 15; ++q) S[15 * k2 + q] = o2[q];
#endif
        }
      }
      // every producer is done reading X[b] before the next iteration gathers tile j + 2's
      // coordinates into it (and before the consumers are released)
      named_sync(5, kGroup);
      named_arrive(1 + b, kAsmThreads);  // buffer b full
    }
    for (int j = (K > 2 ? K - 2 : 0); j < K; ++j) named_sync(3 + (j & 1), kAsmThreads);  // match the last frees
    return;
  }
  for (int j = 0; j < K; ++j) {
    const int b = j & 1;
    named_sync(1 + b, kAsmThreads);
    const unsigned char* blob = blob_of(j);
    const double* S = Sb + b * (kSRecBytes / 8);
    const TileHdr h = *reinterpret_cast<const TileHdr*>(blob);
    const TileLayout L(h.nrows, h.nverts, h.ndom, h.ntask, h.nent);
    const TileRow* rows = reinterpret_cast<const TileRow*>(blob + L.o_rows);
    const TileTask* tasks = reinterpret_cast<const TileTask*>(blob + L.o_task);
    const uint16_t* ent = reinterpret_cast<const uint16_t*>(blob + L.o_ent);
    for (int a = gt; a < (FSFEM_ASM_SKIP == 2 ? 0 : h.ntask); a += kGroup) {
      const TileTask tk = tasks[a];
      double M[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) M[q] = 0.0;
      int e = tk.estart;
      if (tk.sub == 255) {  // off-diagonal block: s_i s_J^T, 6 doubles per entry
#pragma unroll 2
        for (int c = 0; c < tk.count; ++c, ++e) {
          const int en = ent[e];
          const int code = en & 31;
          const int pi = code / 5, pj = code - 5 * pi;
#if FSFEM_ASM_SPLIT
          const double2* SA = reinterpret_cast<const double2*>(S);
          const double* SB = S + 10 * kMaxDom;
          const int kd = 5 * (en >> 5);
          const double2 axy = SA[kd + pi], cxy = SA[kd + pj];
          const double a0 = axy.x, a1 = axy.y, a2 = SB[kd + pi];
          const double c0 = cxy.x, c1 = cxy.y, c2 = SB[kd + pj];
#else
          const double* sd = S + 15 * (en >> 5);
          const double a0 = sd[3 * pi], a1 = sd[3 * pi + 1], a2 = sd[3 * pi + 2];
          const double c0 = sd[3 * pj], c1 = sd[3 * pj + 1], c2 = sd[3 * pj + 2];
#endif
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
      } else {  // diagonal sub-list: s_i s_i^T, 3 doubles per entry (upper triangle)
#pragma unroll 2
        for (int c = 0; c < tk.count; ++c, e += kDiagSplit) {
          const int en = ent[e];
          const int pi = (en & 31) / 6;  // code = 5 pi + pi
#if FSFEM_ASM_SPLIT
          const int kd = 5 * (en >> 5) + pi;
          const double2 axy = reinterpret_cast<const double2*>(S)[kd];
          const double a0 = axy.x, a1 = axy.y, a2 = (S + 10 * kMaxDom)[kd];
#else
          const double* sd = S + 15 * (en >> 5) + 3 * pi;
          const double a0 = sd[0], a1 = sd[1], a2 = sd[2];
#endif
          M[0] = fma(a0, a0, M[0]);
          M[1] = fma(a0, a1, M[1]);
          M[2] = fma(a0, a2, M[2]);
          M[4] = fma(a1, a1, M[4]);
          M[5] = fma(a1, a2, M[5]);
          M[8] = fma(a2, a2, M[8]);
        }
      }
      if (tk.sub == 255) {
        mform_block_store(M, lam, mu, vals + 9 * (rows[tk.row].P + tk.slot));
      } else {  // diagonal sub-list: the 6 independent entries of the symmetric partial
        double* dp = dpart + 6 * (kDiagSplit * tk.row + tk.sub);
        dp[0] = M[0];
        dp[1] = M[4];
        dp[2] = M[8];
        dp[3] = M[1];
        dp[4] = M[2];
        dp[5] = M[5];
      }
    }
    named_sync(6, kGroup);
    if (gt < h.nrows && rows[gt].sdiag >= 0) {  // diagonal blocks: sub-list sums in order
      const int r = gt;
      double d[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      for (int q = 0; q < kDiagSplit; ++q)
#pragma unroll
        for (int v = 0; v < 6; ++v) d[v] += dpart[6 * (kDiagSplit * r + q) + v];
      const double Md[9] = {d[0], d[3], d[4], d[3], d[1], d[5], d[4], d[5], d[2]};
      mform_block_store(Md, lam, mu, vals + 9 * (rows[r].P + rows[r].sdiag));
    }
    named_sync(6, kGroup);              // dpart reused by the next tile
    named_arrive(3 + b, kAsmThreads);   // buffer b free (S, X and the blob slot of tile j)
  }
}

}  // namespace

void face_s_device(const double* xyz, const int32_t* tets, const int32_t* face_nodes, const int32_t* face_tet,
                   const int32_t* face_opp, int64_t nf, double* face_s, double* face_V, cudaStream_t s) {
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nf, 256), 16LL * num_sms())));
  k_face_s<<<grid, 256, 0, s>>>(xyz, tets, face_nodes, face_tet, face_opp, nf, face_s, face_V);
  FS_LAUNCH_CHECK();
}

void tet_s_device(const double* xyz, const int32_t* tets, int64_t nt, double* tet_s, double* tet_V, cudaStream_t s) {
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nt, 256), 16LL * num_sms())));
  k_tet_s<<<grid, 256, 0, s>>>(xyz, tets, nt, tet_s, tet_V);
  FS_LAUNCH_CHECK();
}

void morton_order_device(const double* d_xyz, int64_t nn, int32_t* iperm, int32_t* perm, DevBuf<unsigned char>& scratch,
                         cudaStream_t s);

// Assembly tiles of the pattern (once per pattern; pattern.cuh).  rec_a / rec_b: FS
// face_nodes / face_opp, FEM-T4 tets / unused.  xyz: node coordinates (the tiles follow a Morton
// curve of the own nodes).  Returns an error word in h_flags[0] (kNoError if fine).
void build_assembly_tiles(Pattern& pat, const double* xyz, const int32_t* rec_a, const int32_t* rec_b, bool tet,
                          DevBuf<unsigned char>& scratch, unsigned long long* h_flags, cudaStream_t s) {
  const int64_t nloc = pat.nloc;
  h_flags[0] = kNoError;
  pat.ntiles = 0;
  pat.tile_blob_bytes = 0;
  if (nloc <= 0) return;
  DevBuf<int32_t>& order = pat.tile_order;
  DevBuf<int32_t>& inv = pat.tile_tmp;
  order.ensure(nloc);
  inv.ensure(nloc);
  PhaseTimer pt(s, "tiles");
  morton_order_device(xyz + 3 * pat.n_lo, nloc, order.get(), inv.get(), scratch, s);
  pt.mark("morton order");
  std::vector<int32_t> ts;
  for (int64_t a = 0; a < nloc; a += kTileRows) ts.push_back(static_cast<int32_t>(a));
  ts.push_back(static_cast<int32_t>(nloc));
  static bool attr = false;
  const int bsmem = kBldSmem;
  if (!attr) {
    FS_CUDA(cudaFuncSetAttribute(k_tile_build, cudaFuncAttributeMaxDynamicSharedMemorySize, bsmem));
    FS_CUDA(cudaFuncSetAttribute(k_asm_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAsmSmem));
    FS_CUDA(cudaFuncSetAttribute(k_asm_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAsmSmem));
    attr = true;
  }
  // Build every tile; a tile over a cap is cut in two (first half in place, second half appended)
  // and only the cut tiles are built again (rare: high-valence rows).
  std::vector<int2> tr;
  for (size_t k = 0; k + 1 < ts.size(); ++k) tr.push_back(make_int2(ts[k], ts[k + 1]));
  DevBuf<int2>& d_tr = pat.tile_range;
  std::vector<int64_t> sz;
  std::vector<int32_t> redo;  // tiles to (re)build; empty: all
  for (;;) {
    const int64_t nt = static_cast<int64_t>(tr.size());
    bool all = redo.empty();
    const int64_t cap = nt + nt / 8 + 64;  // room for cut tiles without a reallocation
    if (pat.tile_bytes.n < static_cast<size_t>(nt) || pat.tile_blob.n < static_cast<size_t>(nt) * kBlobCap) {
      pat.tile_bytes.ensure(cap);
      pat.tile_blob.ensure(cap * static_cast<int64_t>(kBlobCap));
      all = true;  // a new allocation holds no built tile
    }
    d_tr.ensure(nt);
    FS_CUDA(cudaMemcpyAsync(d_tr.get(), tr.data(), sizeof(int2) * nt, cudaMemcpyHostToDevice, s));
    const int32_t* which = nullptr;
    int64_t nwork = nt;
    if (!all) {
      pat.tile_redo.ensure(redo.size());
      FS_CUDA(cudaMemcpyAsync(pat.tile_redo.get(), redo.data(), sizeof(int32_t) * redo.size(), cudaMemcpyHostToDevice,
                              s));
      which = pat.tile_redo.get();
      nwork = static_cast<int64_t>(redo.size());
    }
    const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nwork, 8LL * num_sms())));
    k_tile_build<<<g, kBldThreads, bsmem, s>>>(order.get(), d_tr.get(), which, nwork, pat.nf_ptr.get(),
                                               pat.nf_idx.get(), rec_a, rec_b, tet, pat.sptr.get(), pat.snbr.get(),
                                               pat.sdiag.get(), pat.n_lo, pat.tile_bytes.get(), pat.tile_blob.get());
    FS_LAUNCH_CHECK();
    sz.resize(nt);
    FS_CUDA(cudaMemcpyAsync(sz.data(), pat.tile_bytes.get(), sizeof(int64_t) * nt, cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaStreamSynchronize(s));
    pt.mark("tile build + D2H sizes");
    std::vector<int32_t> built;
    if (all) {
      built.resize(nt);
      for (int64_t k = 0; k < nt; ++k) built[k] = static_cast<int32_t>(k);
    } else {
      built.swap(redo);
    }
    redo.clear();
    for (const int32_t k : built) {
      if (sz[k] == -2) {  // one row whose domains exceed the tile caps
        int32_t hord = 0;
        FS_CUDA(cudaMemcpy(&hord, order.get() + tr[k].x, sizeof(int32_t), cudaMemcpyDeviceToHost));
        h_flags[0] = (static_cast<unsigned long long>(FSFEM_ERR_UNSUPPORTED) << 56) |
                     static_cast<unsigned long long>(pat.n_lo + hord);
        return;
      }
      if (sz[k] == -1) {
        const int mid = (tr[k].x + tr[k].y) / 2;
        tr.push_back(make_int2(mid, tr[k].y));
        tr[k].y = mid;
        redo.push_back(k);
        redo.push_back(static_cast<int32_t>(tr.size() - 1));
      }
    }
    if (redo.empty()) break;
  }
  const int64_t nt = static_cast<int64_t>(tr.size());
  int64_t tot = 0, mx = 0;
  for (int64_t k = 0; k < nt; ++k) {
    tot += sz[k];
    mx = std::max(mx, sz[k]);
  }
  pt.mark("host tile sizes");
  pat.ntiles = nt;
  pat.tile_blob_max = mx;
  pat.tile_blob_bytes = tot;
}

// Numeric assembly of the own rows into the stored blocks (S2-S4 + S6).
void assemble_tiles_device(const Pattern& pat, const double* xyz, double lam, double mu, double* vals, bool tet,
                           cudaStream_t s) {
  if (pat.ntiles <= 0) return;
  static int per_sm = 0;
  if (per_sm == 0) {
    FS_CUDA(cudaFuncSetAttribute(k_asm_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAsmSmem));
    FS_CUDA(cudaFuncSetAttribute(k_asm_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAsmSmem));
    FS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_tile<false>, kAsmThreads, kAsmSmem));
    per_sm = std::max(1, per_sm);
  }
  const int g = static_cast<int>(std::min<int64_t>(pat.ntiles, static_cast<int64_t>(per_sm) * num_sms()));
  auto k = tet ? k_asm_tile<true> : k_asm_tile<false>;
  k<<<g, kAsmThreads, kAsmSmem, s>>>(pat.tile_bytes.get(), pat.tile_blob.get(), pat.ntiles, xyz, lam, mu, vals);
  FS_LAUNCH_CHECK();
}

// K7 debug export (fsfem_domain_stiffness): ids, K [n][15][15] and field [n][5] on the device.
void domain_stiffness_device(const double* xyz, const int32_t* rec_a, const int32_t* rec_b, bool tet,
                             const int64_t* ids, int64_t n, double lam, double mu, double* K, int32_t* field,
                             cudaStream_t s) {
  if (n <= 0) return;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 128), 16LL * num_sms())));
  if (tet)
    k_domain_stiffness<true><<<grid, 128, 0, s>>>(xyz, rec_a, rec_b, ids, n, lam, mu, K, field);
  else
    k_domain_stiffness<false><<<grid, 128, 0, s>>>(xyz, rec_a, rec_b, ids, n, lam, mu, K, field);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
