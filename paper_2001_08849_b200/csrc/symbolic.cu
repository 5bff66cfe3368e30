// S5 — symbolic CSR (the pattern of PAPER.md:449 sparse(), built before any value exists).
//
// Node graph of FS-FEM: j is a neighbour of i iff some smoothing domain (face) has both in its
// field.  The field of face f is nodes(t0) U nodes(t1), so the faces whose field holds i are
// exactly the faces of the tets containing i, and
//     nbr(i) = U_{t ni i} ( nodes(t) U { node across each interior face of t } ).
// Every neighbour pair is a dense 3x3 block (Q13): public rows 3i..3i+2 have 3*deg(i) entries.
// Internally only the symmetric half is stored (pattern.cuh): per own node the blocks j >= i
// (plus halo columns j < n_lo), block-contiguous, and a list locating the transposed blocks.
// Per own node we also keep F(i) = the ascending list of faces whose field holds i (the
// summation order of the numeric assembly).
#include <vector>

#include "common.cuh"
#include "pattern.cuh"

namespace fsfem {

namespace {

constexpr int kPatWarps = 4;
constexpr int kMaxTetsPerNode = 128;                 // UNSUPPORTED beyond (general meshes: ~20-60)
constexpr int kCandCap = 8 * kMaxTetsPerNode;        // node candidates per node
constexpr int kFastTetCap = 64;                      // tets per node of the fast pattern pass
constexpr int kPadDeg = 64;  // padded pattern lists of pass 1 (longer lists: a second pattern pass)
constexpr int kSentinel = 0x7fffffff;

__global__ void k_count_node_tets(const int32_t* __restrict__ tets, int64_t nt4, int64_t n_lo, int64_t n_hi,
                                  int32_t* __restrict__ cnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nt4; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = tets[k];
    if (v >= n_lo && v < n_hi) atomicAdd(&cnt[v - n_lo], 1);
  }
}

__global__ void k_scatter_node_tets(const int32_t* __restrict__ tets, int64_t nt4, int64_t n_lo, int64_t n_hi,
                                    const int32_t* __restrict__ ptr, int32_t* __restrict__ cur,
                                    int32_t* __restrict__ idx) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nt4; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = tets[k];
    if (v >= n_lo && v < n_hi) idx[ptr[v - n_lo] + atomicAdd(&cur[v - n_lo], 1)] = static_cast<int32_t>(k >> 2);
  }
}

// Distinct values of src[0..n) (kSentinel entries ignored), ascending, written back to the front
// of src; returns their number.  Warp-wide.  The duplicates are removed first with an open-
// addressing hash set in dst (the order of insertion does not matter: only set membership is
// used), then the few distinct values are ranked (all distinct, so ranks are unique).
// dst is scratch of capacity kCandCap.
__device__ __forceinline__ int warp_sort_unique(int32_t* src, int32_t* dst, int n, int lane, int cap = kCandCap) {
  int H = 64;
  while (H < 2 * n && H < cap) H <<= 1;
  for (int i = lane; i < H; i += 32) dst[i] = kSentinel;
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    const int32_t v = src[i];
    if (v == kSentinel) continue;
    unsigned h = (static_cast<unsigned>(v) * 2654435761u) & (H - 1);
    while (true) {
      const int32_t old = atomicCAS(&dst[h], kSentinel, v);
      if (old == kSentinel || old == v) break;
      h = (h + 1) & (H - 1);
    }
  }
  __syncwarp();
  int count = 0;
  for (int c0 = 0; c0 < H; c0 += 32) {
    const int32_t v = dst[c0 + lane];
    const bool keep = v != kSentinel;
    const unsigned ball = __ballot_sync(0xffffffffu, keep);
    if (keep) src[count + __popc(ball & ((1u << lane) - 1u))] = v;
    count += __popc(ball);
  }
  __syncwarp();
  if (count <= 64) {  // bitonic network in registers: element 2 lane + k, padded with kSentinel
    int32_t a0 = 2 * lane < count ? src[2 * lane] : kSentinel;
    int32_t a1 = 2 * lane + 1 < count ? src[2 * lane + 1] : kSentinel;
#pragma unroll
    for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
      for (int j = size >> 1; j > 0; j >>= 1) {
        if (j == 1) {
          const bool up = ((2 * lane) & size) == 0;
          const int32_t lo = min(a0, a1), hi = max(a0, a1);
          a0 = up ? lo : hi;
          a1 = up ? hi : lo;
        } else {
          const int32_t b0 = __shfl_xor_sync(0xffffffffu, a0, j >> 1);
          const int32_t b1 = __shfl_xor_sync(0xffffffffu, a1, j >> 1);
          const bool lower = ((2 * lane) & j) == 0, up = ((2 * lane) & size) == 0;
          a0 = lower == up ? min(a0, b0) : max(a0, b0);
          a1 = lower == up ? min(a1, b1) : max(a1, b1);
        }
      }
    }
    __syncwarp();
    if (2 * lane < count) src[2 * lane] = a0;
    if (2 * lane + 1 < count) src[2 * lane + 1] = a1;
    __syncwarp();
    return count;
  }
  for (int i = lane; i < count; i += 32) {  // longer lists: rank sort (values are distinct)
    const int32_t v = src[i];
    int r = 0;
    for (int j = 0; j < count; ++j) r += src[j] < v ? 1 : 0;
    dst[r] = v;
  }
  __syncwarp();
  for (int i = lane; i < count; i += 32) src[i] = dst[i];
  __syncwarp();
  return count;
}

// Warp per own node.  Pass 1 (kWrite = false) counts deg(i) and |F(i)|; pass 2 writes the
// sorted lists at node_ptr / nf_ptr and the diagonal slot.  kTetCap = tets per node the shared
// scratch holds: the fast pass-1 instance (64) leaves twice as many warps resident as the full one
// (kMaxTetsPerNode); a node beyond it sets bit 1 of *pad_over and the host reruns pass 1 in full.
template <bool kWrite, int kTetCap = kMaxTetsPerNode>
__global__ void __launch_bounds__(kPatWarps * 32) k_node_pattern(
    const int32_t* __restrict__ tets, const int32_t* __restrict__ tet_face, const int32_t* __restrict__ tet_across,
    const int32_t* __restrict__ nt_ptr, const int32_t* __restrict__ nt_idx,
    int64_t n_lo, int64_t nloc, int32_t* __restrict__ deg, int32_t* __restrict__ nfc,
    const int64_t* __restrict__ node_ptr, const int64_t* __restrict__ nf_ptr, int32_t* __restrict__ nbr,
    int32_t* __restrict__ nf_idx, int32_t* __restrict__ diag_slot, unsigned long long* __restrict__ err, int fem,
    int32_t* __restrict__ pad_nbr, int32_t* __restrict__ pad_nf, int* __restrict__ pad_over) {
  static_assert(kTetCap <= kMaxTetsPerNode, "scratch cap");
  constexpr int kCap = 8 * kTetCap;
  __shared__ int32_t cand[kPatWarps][kCap], tmp[kPatWarps][kCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t il = blockIdx.x * (int64_t)kPatWarps + w; il < nloc; il += (int64_t)gridDim.x * kPatWarps) {
    const int32_t b = nt_ptr[il];
    const int ntet = nt_ptr[il + 1] - b;
    if (ntet > kTetCap) {
      if (lane == 0) {
        if (ntet > kMaxTetsPerNode) report_error(err, FSFEM_ERR_UNSUPPORTED, n_lo + il);
        else if (pad_over != nullptr) atomicOr(pad_over, 2);  // rerun with the full scratch
      }
      continue;
    }
    // candidates: 4 vertices + 4 across-face nodes per tet (the vertex of the neighbour tet
    // opposite face l, from the face table; -1 on the boundary)
    for (int k = lane; k < ntet; k += 32) {
      const int32_t t = nt_idx[b + k];
      const int4 v = reinterpret_cast<const int4*>(tets)[t];
      cand[w][8 * k + 0] = v.x;
      cand[w][8 * k + 1] = v.y;
      cand[w][8 * k + 2] = v.z;
      cand[w][8 * k + 3] = v.w;
      const int4 o = reinterpret_cast<const int4*>(tet_across)[t];
      const bool cpl = !fem;  // FEM-T4 couples only the nodes of a tet
      cand[w][8 * k + 4] = cpl && o.x >= 0 ? o.x : kSentinel;
      cand[w][8 * k + 5] = cpl && o.y >= 0 ? o.y : kSentinel;
      cand[w][8 * k + 6] = cpl && o.z >= 0 ? o.z : kSentinel;
      cand[w][8 * k + 7] = cpl && o.w >= 0 ? o.w : kSentinel;
    }
    __syncwarp();
    const int dn = warp_sort_unique(cand[w], tmp[w], 8 * ntet, lane, kCap);
    if (!kWrite) {
      if (lane == 0) deg[il] = dn;
      if (pad_nbr != nullptr) {  // the sorted list at a fixed stride: pass 2 becomes a copy
        if (dn > kPadDeg) {
          if (lane == 0) atomicOr(pad_over, 1);
        } else {
          for (int k = lane; k < dn; k += 32) pad_nbr[il * kPadDeg + k] = cand[w][k];
        }
      }
    } else {
      const int64_t P = node_ptr[il];
      const int32_t self = static_cast<int32_t>(n_lo + il);
      for (int k = lane; k < dn; k += 32) {
        const int32_t j = cand[w][k];
        nbr[P + k] = j;
        if (j == self) diag_slot[il] = k;
      }
    }
    __syncwarp();
    // FS: faces whose field holds i = the 4 faces of every tet containing i (shared ones twice);
    // FEM-T4: the tets containing i (already ascending).  Either is the assembly order of row i.
    int fn = ntet;
    if (fem) {
      for (int k = lane; k < ntet; k += 32) cand[w][k] = nt_idx[b + k];
      __syncwarp();
    } else {
      for (int k = lane; k < ntet; k += 32) {
        const int32_t t = nt_idx[b + k];
#pragma unroll
        for (int l = 0; l < 4; ++l) cand[w][4 * k + l] = tet_face[4 * t + l];
      }
      __syncwarp();
      fn = warp_sort_unique(cand[w], tmp[w], 4 * ntet, lane, kCap);
    }
    if (!kWrite) {
      if (lane == 0) nfc[il] = fn;
      if (pad_nf != nullptr) {
        if (fn > kPadDeg) {
          if (lane == 0) atomicOr(pad_over, 1);
        } else {
          for (int k = lane; k < fn; k += 32) pad_nf[il * kPadDeg + k] = cand[w][k];
        }
      }
    } else {
      const int64_t Q = nf_ptr[il];
      for (int k = lane; k < fn; k += 32) nf_idx[Q + k] = cand[w][k];
    }
    __syncwarp();
  }
}

// Pass 2 from the padded lists of pass 1: warp per node, copy to the packed offsets.
__global__ void k_pattern_compact(const int32_t* __restrict__ pad_nbr, const int32_t* __restrict__ pad_nf,
                                  int64_t n_lo, int64_t nloc, const int64_t* __restrict__ node_ptr,
                                  const int64_t* __restrict__ nf_ptr, int32_t* __restrict__ nbr,
                                  int32_t* __restrict__ nf_idx, int32_t* __restrict__ diag_slot) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarp = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t il = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); il < nloc; il += nwarp) {
    const int64_t P = node_ptr[il], dn = node_ptr[il + 1] - P;
    const int32_t self = static_cast<int32_t>(n_lo + il);
    for (int k = lane; k < dn; k += 32) {
      const int32_t j = pad_nbr[il * kPadDeg + k];
      nbr[P + k] = j;
      if (j == self) diag_slot[il] = k;
    }
    const int64_t Q = nf_ptr[il], fn = nf_ptr[il + 1] - Q;
    for (int k = lane; k < fn; k += 32) nf_idx[Q + k] = pad_nf[il * kPadDeg + k];
  }
}

// Warp per segment: sort the tets of each node ascending (the atomic scatter left them in
// arbitrary order).  Values in a segment are distinct.
__global__ void __launch_bounds__(kPatWarps * 32) k_sort_segments(const int32_t* __restrict__ ptr, int64_t nseg,
                                                                  int32_t* __restrict__ idx,
                                                                  unsigned long long* __restrict__ err) {
  __shared__ int32_t a[kPatWarps][kMaxTetsPerNode], o[kPatWarps][kMaxTetsPerNode];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t s = blockIdx.x * (int64_t)kPatWarps + w; s < nseg; s += (int64_t)gridDim.x * kPatWarps) {
    const int32_t b = ptr[s];
    const int n = ptr[s + 1] - b;
    if (n > kMaxTetsPerNode) {
      if (lane == 0) report_error(err, FSFEM_ERR_UNSUPPORTED, s);
      continue;
    }
    for (int i = lane; i < n; i += 32) a[w][i] = idx[b + i];
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const int32_t v = a[w][i];
      int r = 0;
      for (int j = 0; j < n; ++j) r += a[w][j] < v ? 1 : 0;
      o[w][r] = v;
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) idx[b + i] = o[w][i];
    __syncwarp();
  }
}

// Symmetric split of every own row (pattern.cuh): count stored (j >= i or j < n_lo) and
// transposed (n_lo <= j < i) blocks.
__global__ void k_split_count(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr, int64_t n_lo,
                              int64_t nloc, int32_t* __restrict__ cnt_s, int32_t* __restrict__ cnt_t) {
  for (int64_t il = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; il < nloc; il += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = n_lo + il;
    int nt = 0;
    for (int64_t k = node_ptr[il]; k < node_ptr[il + 1]; ++k) {
      const int32_t j = nbr[k];
      nt += (j >= n_lo && j < i) ? 1 : 0;
    }
    cnt_t[il] = nt;
    cnt_s[il] = static_cast<int32_t>(node_ptr[il + 1] - node_ptr[il]) - nt;
  }
}

__global__ void k_split_stored(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr, int64_t n_lo,
                               int64_t nloc, const int64_t* __restrict__ sptr, int32_t* __restrict__ snbr,
                               int32_t* __restrict__ sdiag) {
  for (int64_t il = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; il < nloc; il += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = n_lo + il;
    int64_t o = sptr[il];
    sdiag[il] = -1;  // a node in no tet has no blocks at all (BCs then report BREAKDOWN)
    for (int64_t k = node_ptr[il]; k < node_ptr[il + 1]; ++k) {
      const int32_t j = nbr[k];
      if (j >= n_lo && j < i) continue;
      if (j == i) sdiag[il] = static_cast<int32_t>(o - sptr[il]);
      snbr[o++] = j;
    }
  }
}

// For n_lo <= j < i, locate block K_ji in row j (binary search of i in the stored list of j).
__global__ void k_split_trans(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr, int64_t n_lo,
                              int64_t nloc, const int64_t* __restrict__ sptr, const int32_t* __restrict__ snbr,
                              const int64_t* __restrict__ tptr, int2* __restrict__ tlist,
                              unsigned long long* __restrict__ err) {
  for (int64_t il = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; il < nloc; il += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = static_cast<int32_t>(n_lo + il);
    int64_t o = tptr[il];
    for (int64_t k = node_ptr[il]; k < node_ptr[il + 1]; ++k) {
      const int32_t j = nbr[k];
      if (!(j >= n_lo && j < i)) continue;
      int64_t lo = sptr[j - n_lo], hi = sptr[j - n_lo + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (snbr[mid] < i) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= sptr[j - n_lo + 1] || snbr[lo] != i) report_error(err, FSFEM_ERR_TOPOLOGY, i);  // asymmetric graph
      tlist[o++] = make_int2(static_cast<int32_t>(lo), j);
    }
  }
}

// Push SpMV support: tpos[b] = slot of stored block b in the transposed list of its column row.
__global__ void k_tpos(const int2* __restrict__ tlist, int64_t ntb, int32_t* __restrict__ tpos) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntb; k += (int64_t)gridDim.x * blockDim.x)
    tpos[tlist[k].x] = static_cast<int32_t>(k);
}

// Warp per chunk c: the distinct chunks d < c that hold a producer row (j of a transposed entry
// (K_ji, j) of the chunk's rows), ascending; more than kMaxDeps -> ndeps = -1 and the waiter
// checks the whole range [deps[0], c).
constexpr int kDepWarps = 4;
__global__ void __launch_bounds__(kDepWarps * 32) k_chunk_deps(const SpmvChunk* __restrict__ ch, int nch,
                                                                const int2* __restrict__ tlist, int64_t n_lo,
                                                                int32_t* __restrict__ deps, int32_t* __restrict__ ndeps) {
  __shared__ int32_t pcs[kDepWarps][kCapBlocks];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = blockIdx.x * kDepWarps + w; c < nch; c += gridDim.x * kDepWarps) {
    const int Pt0 = ch[c].Pt0, n = ch[c].Pt1 - Pt0;
    for (int k = lane; k < n; k += 32) {
      const int32_t j = static_cast<int32_t>(tlist[Pt0 + k].y - n_lo);
      int lo = 0, hi = c;  // last chunk d <= c with ch[d].n0 <= j
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ch[mid].n0 <= j) lo = mid;
        else hi = mid - 1;
      }
      pcs[w][k] = lo;
    }
    __syncwarp();
    int last = -1, cnt = 0;
    while (cnt <= kMaxDeps) {
      int m = 0x7fffffff;
      for (int k = lane; k < n; k += 32) {
        const int v = pcs[w][k];
        if (v < c && v > last) m = min(m, v);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (m == 0x7fffffff) break;
      if (lane == 0 && cnt < kMaxDeps) deps[static_cast<int64_t>(c) * kMaxDeps + cnt] = m;
      ++cnt;
      last = m;
    }
    if (lane == 0) ndeps[c] = cnt <= kMaxDeps ? cnt : -1;
    __syncwarp();
  }
}

// SpMV streaming chunks (pattern.cuh), built on the device: windows of kChunkNodes own nodes
// (aligned to the rank's first node); a window whose stored or transposed block count exceeds
// kCapBlocks is cut greedily into runs that fit (high-valence rows).  out == nullptr: count only.
// Returns -1 when one node alone exceeds kCapBlocks.
__device__ int window_chunks(const int64_t* __restrict__ sptr, const int64_t* __restrict__ tptr, int64_t a, int64_t b,
                             SpmvChunk* out, int64_t* bad_node) {
  int n = 0;
  for (int64_t n0 = a; n0 < b;) {
    int64_t n1 = n0;
    while (n1 < b && sptr[n1 + 1] - sptr[n0] <= kCapBlocks && tptr[n1 + 1] - tptr[n0] <= kCapBlocks) ++n1;
    if (n1 == n0) {
      *bad_node = n0;
      return -1;
    }
    if (out)
      out[n] = SpmvChunk{static_cast<int32_t>(n0), static_cast<int32_t>(n1), static_cast<int32_t>(sptr[n0]),
                         static_cast<int32_t>(sptr[n1]), static_cast<int32_t>(tptr[n0]), static_cast<int32_t>(tptr[n1]),
                         0, 0};
    ++n;
    n0 = n1;
  }
  return n;
}

__global__ void k_chunk_count(const int64_t* __restrict__ sptr, const int64_t* __restrict__ tptr, int64_t nloc,
                              int64_t n_lo, int32_t* __restrict__ cnt, unsigned long long* __restrict__ err) {
  const int64_t nw = (nloc + kChunkNodes - 1) / kChunkNodes;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t bad = 0;
    const int n = window_chunks(sptr, tptr, w * kChunkNodes, min(nloc, (w + 1) * kChunkNodes), nullptr, &bad);
    if (n < 0) report_error(err, FSFEM_ERR_UNSUPPORTED, n_lo + bad);
    cnt[w] = max(n, 0);
  }
}

__global__ void k_chunk_emit(const int64_t* __restrict__ sptr, const int64_t* __restrict__ tptr, int64_t nloc,
                             const int32_t* __restrict__ off, SpmvChunk* __restrict__ chunks) {
  const int64_t nw = (nloc + kChunkNodes - 1) / kChunkNodes;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t bad = 0;
    window_chunks(sptr, tptr, w * kChunkNodes, min(nloc, (w + 1) * kChunkNodes), chunks + off[w], &bad);
  }
}

// Reverse producer lists of the dataflow SpMV: for every chunk d the chunks c that need it (d
// itself and every c with d among its producers), each with its need ndeps[c] + 1, ascending c.
// A chunk with more than kMaxDeps producers (ndeps = -1) disables the dataflow kernel (*bad).
__global__ void k_rdeps_count(const int32_t* __restrict__ ndeps, const int32_t* __restrict__ deps, int nch,
                              int32_t* __restrict__ cnt, unsigned long long* __restrict__ bad) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += gridDim.x * blockDim.x) {
    const int nd = ndeps[c];
    if (nd < 0) {
      atomicExch(bad, 1ull);
      continue;
    }
    atomicAdd(cnt + c, 1);
    for (int k = 0; k < nd; ++k) atomicAdd(cnt + deps[static_cast<int64_t>(c) * kMaxDeps + k], 1);
  }
}

__global__ void k_rdeps_fill(const int32_t* __restrict__ ndeps, const int32_t* __restrict__ deps, int nch,
                             const int32_t* __restrict__ ptr, int32_t* __restrict__ cur, int2* __restrict__ tmp) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += gridDim.x * blockDim.x) {
    const int nd = ndeps[c];
    if (nd < 0) continue;
    const int2 e = make_int2(c, nd + 1);
    tmp[ptr[c] + atomicAdd(cur + c, 1)] = e;
    for (int k = 0; k < nd; ++k) {
      const int d = deps[static_cast<int64_t>(c) * kMaxDeps + k];
      tmp[ptr[d] + atomicAdd(cur + d, 1)] = e;
    }
  }
}

// Warp per list: rank by consumer chunk (distinct within a list) into the final order.
__global__ void k_rdeps_sort(const int32_t* __restrict__ ptr, int nch, const int2* __restrict__ tmp,
                             int2* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarp = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t d = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); d < nch; d += nwarp) {
    const int a = ptr[d], n = ptr[d + 1] - a;
    for (int i = lane; i < n; i += 32) {
      const int2 e = tmp[a + i];
      int r = 0;
      for (int j = 0; j < n; ++j) r += tmp[a + j].x < e.x ? 1 : 0;
      list[a + r] = e;
    }
  }
}

// Expand the symmetric block storage to the public CSR (row_ptr int64, col_idx int32, vals):
// row 3i+a lists columns 3j+c for j in nbr(i) ascending.  In nbr order a row is
// [halo stored (j < n_lo)] [transposed (n_lo <= j < i)] [stored j >= i]; the diagonal is the
// first non-halo stored block, so the halo count equals sdiag.
__global__ void k_export_csr(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr,
                             const int64_t* __restrict__ sptr, const int32_t* __restrict__ sdiag,
                             const int64_t* __restrict__ tptr, const int2* __restrict__ tlist,
                             const double* __restrict__ svals, int64_t nloc, int64_t* __restrict__ row_ptr,
                             int32_t* __restrict__ col_idx, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  for (int64_t il = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; il < nloc;
       il += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t P = node_ptr[il];
    const int deg = static_cast<int>(node_ptr[il + 1] - P);
    const int m = 3 * deg;
    const int h = sdiag[il];
    const int ntr = static_cast<int>(tptr[il + 1] - tptr[il]);
    if (row_ptr && lane < 3) row_ptr[3 * il + lane] = 9 * P + lane * m;
    if (row_ptr && il == nloc - 1 && lane == 0) row_ptr[3 * nloc] = 9 * node_ptr[nloc];
    for (int s = lane; s < deg; s += 32) {
      const int32_t j = nbr[P + s];
      if (col_idx) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) col_idx[9 * P + a * m + 3 * s + c] = 3 * j + c;
      }
      if (!vals) continue;
      double blk[9];
      if (s >= h && s < h + ntr) {
        const double* src = svals + 9 * static_cast<int64_t>(tlist[tptr[il] + (s - h)].x);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) blk[3 * a + c] = src[3 * c + a];
      } else {
        const double* src = svals + 9 * (sptr[il] + (s < h ? s : s - ntr));
#pragma unroll
        for (int q = 0; q < 9; ++q) blk[q] = src[q];
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) vals[9 * P + a * m + 3 * s + c] = blk[3 * a + c];
    }
  }
}

}  // namespace

// Host driver of S5 for the own node range [n_lo, n_lo + nloc).
void build_pattern_device(const int32_t* d_tets, int64_t nt, const int32_t* tet_face, const int32_t* tet_across,
                          int64_t n_lo, int64_t nloc, cudaStream_t s,
                          DevBuf<unsigned char>& scratch, Pattern& pat, unsigned long long* h_flags, int fem) {
  DevBuf<int64_t>& node_ptr = pat.node_ptr;
  DevBuf<int32_t>& nbr = pat.nbr;
  DevBuf<int64_t>& nf_ptr = pat.nf_ptr;
  DevBuf<int32_t>& nf_idx = pat.nf_idx;
  DevBuf<int32_t>& diag_slot = pat.diag_full;
  pat.n_lo = n_lo;
  pat.nloc = nloc;
  const int sms = num_sms();
  size_t o = 0;
  auto carve = [&](size_t bytes) {
    size_t at = o;
    o += (bytes + 255) & ~size_t(255);
    return at;
  };
  const size_t o_cnt = carve(sizeof(int32_t) * (nloc + 1));
  const size_t o_ptr = carve(sizeof(int32_t) * (nloc + 1));
  const size_t o_cur = carve(sizeof(int32_t) * (nloc + 1));
  const size_t o_idx = carve(sizeof(int32_t) * 4 * nt);
  const size_t o_deg = carve(sizeof(int32_t) * (nloc + 1));
  const size_t o_nfc = carve(sizeof(int32_t) * (nloc + 1));
  const size_t o_flags = carve(sizeof(unsigned long long) * 2);
  const size_t o_tmp = carve(scan_tmp_bytes(nloc + 1));
  const size_t o_pad = carve(sizeof(int32_t) * 2 * kPadDeg * std::max<int64_t>(nloc, 1) + 16);
  unsigned char* base = scratch.ensure(o);
  int32_t* cnt = reinterpret_cast<int32_t*>(base + o_cnt);
  int32_t* ptr = reinterpret_cast<int32_t*>(base + o_ptr);
  int32_t* cur = reinterpret_cast<int32_t*>(base + o_cur);
  int32_t* idx = reinterpret_cast<int32_t*>(base + o_idx);
  int32_t* deg = reinterpret_cast<int32_t*>(base + o_deg);
  int32_t* nfc = reinterpret_cast<int32_t*>(base + o_nfc);
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(base + o_flags);
  void* tmp = base + o_tmp;
  const size_t tb = scan_tmp_bytes(nloc + 1);
  int32_t* pad_nbr = reinterpret_cast<int32_t*>(base + o_pad);
  int32_t* pad_nf = pad_nbr + kPadDeg * nloc;
  int* pad_over = reinterpret_cast<int*>(pad_nf + kPadDeg * nloc);

  PhaseTimer pt(s, "symbolic");
  FS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nloc + 1), s));
  FS_CUDA(cudaMemsetAsync(cur, 0, sizeof(int32_t) * (nloc + 1), s));
  FS_CUDA(cudaMemsetAsync(flags, 0xff, sizeof(unsigned long long), s));
  FS_CUDA(cudaMemsetAsync(pad_over, 0, sizeof(int), s));
  const int g4 = static_cast<int>(std::min<int64_t>(ceil_div(4 * nt, 256), 8LL * sms));
  k_count_node_tets<<<g4, 256, 0, s>>>(d_tets, 4 * nt, n_lo, n_lo + nloc, cnt);
  FS_LAUNCH_CHECK();
  exclusive_scan_i32(cnt, ptr, nloc, s, tmp, tb);
  k_scatter_node_tets<<<g4, 256, 0, s>>>(d_tets, 4 * nt, n_lo, n_lo + nloc, ptr, cur, idx);
  FS_LAUNCH_CHECK();
  const int gw = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, kPatWarps), 32LL * sms)));
  k_sort_segments<<<gw, kPatWarps * 32, 0, s>>>(ptr, nloc, idx, flags);
  FS_LAUNCH_CHECK();
  pt.mark("node tets");
  k_node_pattern<false, kFastTetCap><<<gw, kPatWarps * 32, 0, s>>>(d_tets, tet_face, tet_across, ptr, idx, n_lo,
                                                                   nloc, deg, nfc, nullptr, nullptr, nullptr, nullptr,
                                                                   nullptr, flags, fem, pad_nbr, pad_nf, pad_over);
  FS_LAUNCH_CHECK();
  node_ptr.ensure(nloc + 1);
  nf_ptr.ensure(nloc + 1);
  int64_t tot[2];
  int h_over = 0;
  auto scan_and_read = [&]() {
    exclusive_scan_i32_to_i64(deg, node_ptr.get(), nloc, s, tmp, tb);
    exclusive_scan_i32_to_i64(nfc, nf_ptr.get(), nloc, s, tmp, tb);
    FS_CUDA(cudaMemcpyAsync(&tot[0], node_ptr.get() + nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaMemcpyAsync(&tot[1], nf_ptr.get() + nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaMemcpyAsync(h_flags, flags, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaMemcpyAsync(&h_over, pad_over, sizeof(int), cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaStreamSynchronize(s));
  };
  scan_and_read();
  if (h_flags[0] == kNoError && (h_over & 2)) {  // a node in more than kFastTetCap tets: full pass 1
    FS_CUDA(cudaMemsetAsync(pad_over, 0, sizeof(int), s));
    k_node_pattern<false><<<gw, kPatWarps * 32, 0, s>>>(d_tets, tet_face, tet_across, ptr, idx, n_lo, nloc, deg,
                                                        nfc, nullptr, nullptr, nullptr, nullptr, nullptr, flags, fem,
                                                        pad_nbr, pad_nf, pad_over);
    FS_LAUNCH_CHECK();
    scan_and_read();
  }
  pt.mark("pattern count + scans");
  if (h_flags[0] != kNoError) return;
  pat.nblk = tot[0];
  pat.nfi = tot[1];
  nbr.ensure(tot[0]);
  nf_idx.ensure(tot[1]);
  diag_slot.ensure(nloc);
  if ((h_over & 1) == 0) {
    k_pattern_compact<<<gw, kPatWarps * 32, 0, s>>>(pad_nbr, pad_nf, n_lo, nloc, node_ptr.get(), nf_ptr.get(), nbr.get(),
                                                    nf_idx.get(), diag_slot.get());
  } else {
    k_node_pattern<true><<<gw, kPatWarps * 32, 0, s>>>(d_tets, tet_face, tet_across, ptr, idx, n_lo, nloc,
                                                       nullptr, nullptr, node_ptr.get(), nf_ptr.get(), nbr.get(),
                                                       nf_idx.get(), diag_slot.get(), flags, fem, nullptr, nullptr,
                                                       nullptr);
  }
  FS_LAUNCH_CHECK();
  pt.mark("pattern write");
  // symmetric split (pattern.cuh): deg and nfc are free again, reuse them as counters
  const int gt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 256), 8LL * sms)));
  k_split_count<<<gt, 256, 0, s>>>(node_ptr.get(), nbr.get(), n_lo, nloc, deg, nfc);
  FS_LAUNCH_CHECK();
  pat.sptr.ensure(nloc + 3);
  pat.tptr.ensure(nloc + 3);
  exclusive_scan_i32_to_i64(deg, pat.sptr.get(), nloc, s, tmp, tb);
  exclusive_scan_i32_to_i64(nfc, pat.tptr.get(), nloc, s, tmp, tb);
  FS_CUDA(cudaMemcpyAsync(&tot[0], pat.sptr.get() + nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaMemcpyAsync(&tot[1], pat.tptr.get() + nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  pat.nsb = tot[0];
  pat.ntb = tot[1];
  pat.snbr.ensure(pat.nsb + 4);  // + slack for the SpMV bulk copies (pattern.cuh)
  pat.sdiag.ensure(std::max<int64_t>(nloc, 1));
  pat.tlist.ensure(pat.ntb + 2);
  k_split_stored<<<gt, 256, 0, s>>>(node_ptr.get(), nbr.get(), n_lo, nloc, pat.sptr.get(), pat.snbr.get(),
                                    pat.sdiag.get());
  FS_LAUNCH_CHECK();
  k_split_trans<<<gt, 256, 0, s>>>(node_ptr.get(), nbr.get(), n_lo, nloc, pat.sptr.get(), pat.snbr.get(),
                                   pat.tptr.get(), pat.tlist.get(), flags);
  FS_LAUNCH_CHECK();
  // SpMV streaming chunks (pattern.cuh): windows of kChunkNodes nodes, split where a window's
  // stored or transposed block count exceeds kCapBlocks
  const int64_t nw = ceil_div(nloc, kChunkNodes);
  const int gc = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nw, 256), 8LL * sms)));
  k_chunk_count<<<gc, 256, 0, s>>>(pat.sptr.get(), pat.tptr.get(), nloc, n_lo, deg, flags);
  FS_LAUNCH_CHECK();
  exclusive_scan_i32(deg, nfc, nw, s, tmp, tb);
  int32_t nch32 = 0;
  FS_CUDA(cudaMemcpyAsync(h_flags, flags, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaMemcpyAsync(&nch32, nfc + nw, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  pt.mark("split + chunk count");
  if (h_flags[0] != kNoError) return;
  pat.nchunks = nch32;
  pat.chunks.ensure(std::max<int64_t>(pat.nchunks, 1));
  k_chunk_emit<<<gc, 256, 0, s>>>(pat.sptr.get(), pat.tptr.get(), nloc, nfc, pat.chunks.get());
  FS_LAUNCH_CHECK();
  // push SpMV: slots of the stored blocks, per-chunk producer lists, fresh flags and epoch
  pat.tpos.ensure(pat.nsb + 4);
  pat.tbuf.ensure(3 * pat.ntb + 2);
  pat.deps.ensure(std::max<int64_t>(pat.nchunks, 1) * kMaxDeps);
  pat.ndeps.ensure(std::max<int64_t>(pat.nchunks, 1));
  pat.cflags.ensure(std::max<int64_t>(pat.nchunks, 1));
  pat.sync.ensure(2);
  FS_CUDA(cudaMemsetAsync(pat.tpos.get(), 0xff, sizeof(int32_t) * (pat.nsb + 4), s));
  FS_CUDA(cudaMemsetAsync(pat.cflags.get(), 0, sizeof(uint32_t) * std::max<int64_t>(pat.nchunks, 1), s));
  FS_CUDA(cudaMemsetAsync(pat.sync.get(), 0, sizeof(uint32_t) * 2, s));
  if (pat.ntb > 0) {
    const int gp = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(pat.ntb, 256), 8LL * sms)));
    k_tpos<<<gp, 256, 0, s>>>(pat.tlist.get(), pat.ntb, pat.tpos.get());
    FS_LAUNCH_CHECK();
  }
  pat.df_ok = false;
  if (pat.nchunks > 0) {
    const int nch = static_cast<int>(pat.nchunks);
    const int gd = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(pat.nchunks, kDepWarps), 16LL * sms)));
    k_chunk_deps<<<gd, kDepWarps * 32, 0, s>>>(pat.chunks.get(), nch, pat.tlist.get(), n_lo, pat.deps.get(),
                                               pat.ndeps.get());
    FS_LAUNCH_CHECK();
    // reverse lists for the dataflow SpMV (deg / nfc reused as counters)
    const int gr = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(pat.nchunks, 256), 8LL * sms)));
    FS_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * (nch + 1), s));
    FS_CUDA(cudaMemsetAsync(flags + 1, 0, sizeof(unsigned long long), s));
    k_rdeps_count<<<gr, 256, 0, s>>>(pat.ndeps.get(), pat.deps.get(), nch, deg, flags + 1);
    FS_LAUNCH_CHECK();
    pat.dep_ptr.ensure(nch + 1);
    exclusive_scan_i32(deg, pat.dep_ptr.get(), nch, s, tmp, tb);
    const int64_t cap = static_cast<int64_t>(nch) * (kMaxDeps + 1);
    pat.dep_list.ensure(cap);
    pat.dep_tmp.ensure(cap);
    FS_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * (nch + 1), s));
    k_rdeps_fill<<<gr, 256, 0, s>>>(pat.ndeps.get(), pat.deps.get(), nch, pat.dep_ptr.get(), deg, pat.dep_tmp.get());
    FS_LAUNCH_CHECK();
    k_rdeps_sort<<<gd, kDepWarps * 32, 0, s>>>(pat.dep_ptr.get(), nch, pat.dep_tmp.get(), pat.dep_list.get());
    FS_LAUNCH_CHECK();
    pat.cnt.ensure(nch);
    pat.dotc.ensure(nch);
    FS_CUDA(cudaMemsetAsync(pat.cnt.get(), 0, sizeof(uint32_t) * nch, s));
    FS_CUDA(cudaMemcpyAsync(h_flags + 3, flags + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaStreamSynchronize(s));
    pat.df_ok = h_flags[3] == 0;
    pt.mark("chunks + tpos + deps");
  }
  FS_CUDA(cudaStreamSynchronize(s));
}

void export_csr_device(const Pattern& pat, const double* svals, int64_t* row_ptr, int32_t* col_idx, double* vals,
                       cudaStream_t s) {
  if (pat.nloc == 0) return;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(pat.nloc * 32, 256), 32LL * num_sms()));
  k_export_csr<<<std::max(grid, 1), 256, 0, s>>>(pat.node_ptr.get(), pat.nbr.get(), pat.sptr.get(), pat.sdiag.get(),
                                                  pat.tptr.get(), pat.tlist.get(), svals, pat.nloc, row_ptr, col_idx,
                                                  vals);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
