// Internal node renumbering for locality (DESIGN.md §5 "node order").
//
// The SpMV and the assembly gather x and face records through L1/L2, so they rely on the node
// numbering being banded (neighbours have nearby ids).  A mesh whose numbering is not (e.g. a
// random relabelling, BASELINE configs[4]) is renumbered internally in Morton order of its node
// coordinates; every API output stays in the caller's numbering.  perm: user -> internal,
// iperm: internal -> user.  Nothing here changes what is computed, only where it is stored.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "pattern.cuh"

namespace fsfem {

namespace {

// Sum over tets of (max id - min id): the numbering's bandwidth (integer sum: exact).
__global__ void k_tet_span(const int4* __restrict__ tets, int64_t nt, unsigned long long* __restrict__ out) {
  unsigned long long s = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = tets[t];
    const int lo = min(min(v.x, v.y), min(v.z, v.w)), hi = max(max(v.x, v.y), max(v.z, v.w));
    s += static_cast<unsigned long long>(hi - lo);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void k_perm_ids(const int32_t* __restrict__ perm, const int32_t* __restrict__ in, int32_t* __restrict__ out,
                           int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = in[k];
    out[k] = v < 0 ? v : perm[v];
  }
}

__global__ void k_perm_ids_valid(const int32_t* __restrict__ perm, const int32_t* __restrict__ in,
                                 int32_t* __restrict__ out, int64_t n, int64_t nn) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = in[k];
    out[k] = (v >= 0 && v < nn) ? perm[v] : v;  // invalid ids stay invalid (reported downstream)
  }
}

// out[w*i + a] = in[w*iperm[i] + a] (to_internal) or out[w*iperm[i] + a] = in[w*i + a].
template <typename T>
__global__ void k_permute_rows(const int32_t* __restrict__ iperm, const T* __restrict__ in, T* __restrict__ out,
                               int64_t nn, int w, bool to_internal) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nn * w; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / w, a = k - i * w;
    const int64_t u = iperm[i];
    if (to_internal) out[k] = in[w * u + a];
    else out[w * u + a] = in[k];
  }
}

// Public CSR in the caller's numbering from the (internally numbered) symmetric storage.
// Warp per user node I: its internal row i = perm[I]; the neighbours are mapped to user ids and
// ranked (ascending user column order), then each lane emits its blocks like k_export_csr.
constexpr int kExpWarps = 4;
constexpr int kExpCap = 1024;
__global__ void __launch_bounds__(kExpWarps * 32) k_export_csr_user(
    const int32_t* __restrict__ perm, const int32_t* __restrict__ iperm, const int64_t* __restrict__ node_ptr,
    const int32_t* __restrict__ nbr, const int64_t* __restrict__ sptr, const int32_t* __restrict__ sdiag,
    const int64_t* __restrict__ tptr, const int2* __restrict__ tlist, const double* __restrict__ svals,
    const int64_t* __restrict__ uptr /* user-order node offsets */, int64_t nn, int64_t* __restrict__ row_ptr,
    int32_t* __restrict__ col_idx, double* __restrict__ vals) {
  __shared__ int32_t ucol[kExpWarps][kExpCap];
  __shared__ int32_t order[kExpWarps][kExpCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t I = blockIdx.x * (int64_t)kExpWarps + w; I < nn; I += (int64_t)gridDim.x * kExpWarps) {
    const int64_t i = perm[I];
    const int64_t P = node_ptr[i];
    const int deg = static_cast<int>(node_ptr[i + 1] - P);
    const int m = 3 * deg;
    const int64_t PU = uptr[I];
    if (row_ptr && lane < 3) row_ptr[3 * I + lane] = 9 * PU + lane * m;
    if (row_ptr && I == nn - 1 && lane == 0) row_ptr[3 * nn] = 9 * uptr[nn];
    for (int s = lane; s < deg; s += 32) ucol[w][s] = iperm[nbr[P + s]];
    __syncwarp();
    for (int s = lane; s < deg; s += 32) {  // rank of each neighbour among the user ids (distinct)
      const int32_t v = ucol[w][s];
      int r = 0;
      for (int t = 0; t < deg; ++t) r += ucol[w][t] < v ? 1 : 0;
      order[w][r] = s;
    }
    __syncwarp();
    const int h = sdiag[i];
    const int ntr = static_cast<int>(tptr[i + 1] - tptr[i]);
    for (int r = lane; r < deg; r += 32) {
      const int s = order[w][r];  // internal slot of the r-th user column
      const int32_t j = ucol[w][s];
      if (col_idx) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) col_idx[9 * PU + a * m + 3 * r + c] = 3 * j + c;
      }
      if (!vals) continue;
      double blk[9];
      if (s >= h && s < h + ntr) {
        const double* src = svals + 9 * static_cast<int64_t>(tlist[tptr[i] + (s - h)].x);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) blk[3 * a + c] = src[3 * c + a];
      } else {
        const double* src = svals + 9 * (sptr[i] + (s < h ? s : s - ntr));
#pragma unroll
        for (int q = 0; q < 9; ++q) blk[q] = src[q];
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) vals[9 * PU + a * m + 3 * r + c] = blk[3 * a + c];
    }
    __syncwarp();
  }
}

__global__ void k_user_degrees(const int32_t* __restrict__ perm, const int64_t* __restrict__ node_ptr, int64_t nn,
                               int64_t* __restrict__ deg) {
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < nn; I += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = perm[I];
    deg[I] = node_ptr[i + 1] - node_ptr[i];
  }
}

int grid_for(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 16LL * num_sms())));
}


// ---- Morton order on the device: 30-bit keys (10 bits per axis over one common cell size), then a
// stable LSD radix sort (4 passes of 8 bits) of (key, node id) starting from id order, so equal
// keys keep ascending ids: the order is a pure function of the coordinates.
__device__ __forceinline__ uint32_t spread3_10(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void k_morton_keys(const double* __restrict__ xyz, int64_t nn, const double* __restrict__ bbox,
                              uint32_t* __restrict__ key, int32_t* __restrict__ val) {
  const double ext = fmax(bbox[3] - bbox[0], fmax(bbox[4] - bbox[1], bbox[5] - bbox[2]));
  const double sc = ext > 0.0 ? 1023.0 / ext : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double q = (xyz[3 * i + a] - bbox[a]) * sc;
      k |= spread3_10(static_cast<uint32_t>(fmin(fmax(q, 0.0), 1023.0))) << a;
    }
    key[i] = k;
    val[i] = static_cast<int32_t>(i);
  }
}

constexpr int kRsThreads = 256, kRsItems = 8, kRsTile = kRsThreads * kRsItems;

// per-tile digit counts, digit-major: hist[d * ntiles + tile]
__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint32_t* __restrict__ key, int64_t n, int shift,
                                                        int32_t* __restrict__ hist, int ntiles) {
  __shared__ int32_t cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
  for (int r = 0; r < kRsItems; ++r) {
    const int64_t i = base + r * kRsThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(key[i] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

// stable scatter: items of a tile in round-major order (index = base + r * 256 + t), ranked by
// warp match + per-warp counts + a running per-digit counter of the tile
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint32_t* __restrict__ key,
                                                           const int32_t* __restrict__ val, int64_t n, int shift,
                                                           const int32_t* __restrict__ off, int ntiles,
                                                           uint32_t* __restrict__ key_out, int32_t* __restrict__ val_out) {
  __shared__ int32_t run[256];
  __shared__ int32_t wcnt[kRsThreads / 32][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  run[threadIdx.x] = off[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
  for (int r = 0; r < kRsItems; ++r) {
    for (int k = threadIdx.x; k < (kRsThreads / 32) * 256; k += kRsThreads) (&wcnt[0][0])[k] = 0;
    __syncthreads();
    const int64_t i = base + r * kRsThreads + threadIdx.x;
    const bool ok = i < n;
    const uint32_t kk = ok ? key[i] : 0u;
    const int32_t vv = ok ? val[i] : 0;
    const int d = ok ? static_cast<int>((kk >> shift) & 255u) : 256 + lane;  // inactive lanes: unique dummies
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (ok && rank == 0) wcnt[w][d] = __popc(peers);
    __syncthreads();
    int before = 0;
    if (ok)
      for (int q = 0; q < w; ++q) before += wcnt[q][d];
    if (ok) {
      const int64_t pos = run[d] + before + rank;
      key_out[pos] = kk;
      val_out[pos] = vv;
    }
    __syncthreads();
    {  // advance the running counters by this round's totals
      int tot = 0;
      for (int q = 0; q < kRsThreads / 32; ++q) tot += wcnt[q][threadIdx.x];
      run[threadIdx.x] += tot;
    }
    __syncthreads();
  }
}

__global__ void k_inverse_perm(const int32_t* __restrict__ iperm, int64_t n, int32_t* __restrict__ perm) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    perm[iperm[k]] = static_cast<int32_t>(k);
}

}  // namespace

void bbox_device(const double* d_xyz, int64_t nn, double* part, double* bbox, cudaStream_t s);

// iperm (internal -> user) and perm (user -> internal) of the Morton order, on the device.
void morton_order_device(const double* d_xyz, int64_t nn, int32_t* iperm, int32_t* perm,
                         DevBuf<unsigned char>& scratch, cudaStream_t s) {
  if (nn <= 0) return;
  const int ntiles = static_cast<int>(ceil_div(nn, kRsTile));
  const int64_t nh = 256LL * ntiles;
  size_t o = 0;
  auto carve = [&](size_t bytes) {
    const size_t at = o;
    o += (bytes + 255) & ~size_t(255);
    return at;
  };
  const size_t o_part = carve(sizeof(double) * 6 * 16 * num_sms()), o_bb = carve(sizeof(double) * 8),
               o_k0 = carve(4 * nn), o_k1 = carve(4 * nn), o_v1 = carve(4 * nn), o_h = carve(4 * (nh + 1)),
               o_off = carve(4 * (nh + 1)), o_tmp = carve(scan_tmp_bytes(nh + 1));
  unsigned char* b = scratch.ensure(o);
  double* part = reinterpret_cast<double*>(b + o_part);
  double* bb = reinterpret_cast<double*>(b + o_bb);
  uint32_t* k0 = reinterpret_cast<uint32_t*>(b + o_k0);
  uint32_t* k1 = reinterpret_cast<uint32_t*>(b + o_k1);
  int32_t* v0 = iperm;  // the values end in iperm after the 4th (even) pass
  int32_t* v1 = reinterpret_cast<int32_t*>(b + o_v1);
  int32_t* hist = reinterpret_cast<int32_t*>(b + o_h);
  int32_t* off = reinterpret_cast<int32_t*>(b + o_off);
  bbox_device(d_xyz, nn, part, bb, s);
  k_morton_keys<<<grid_for(nn), 256, 0, s>>>(d_xyz, nn, bb, k0, v0);
  FS_LAUNCH_CHECK();
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 8 * pass;
    uint32_t* kin = (pass & 1) ? k1 : k0;
    uint32_t* kout = (pass & 1) ? k0 : k1;
    int32_t* vin = (pass & 1) ? v1 : v0;
    int32_t* vout = (pass & 1) ? v0 : v1;
    k_rs_hist<<<ntiles, kRsThreads, 0, s>>>(kin, nn, shift, hist, ntiles);
    FS_LAUNCH_CHECK();
    exclusive_scan_i32(hist, off, nh, s, b + o_tmp, scan_tmp_bytes(nh + 1));
    k_rs_scatter<<<ntiles, kRsThreads, 0, s>>>(kin, vin, nn, shift, off, ntiles, kout, vout);
    FS_LAUNCH_CHECK();
  }
  k_inverse_perm<<<grid_for(nn), 256, 0, s>>>(iperm, nn, perm);
  FS_LAUNCH_CHECK();
}

// Mean tet id span (user numbering), exact.
double mean_tet_span_device(const int32_t* tets, int64_t nt, unsigned long long* d_tmp, cudaStream_t s) {
  FS_CUDA(cudaMemsetAsync(d_tmp, 0, sizeof(unsigned long long), s));
  k_tet_span<<<grid_for(nt), 256, 0, s>>>(reinterpret_cast<const int4*>(tets), nt, d_tmp);
  FS_LAUNCH_CHECK();
  unsigned long long h = 0;
  FS_CUDA(cudaMemcpyAsync(&h, d_tmp, sizeof(h), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  return static_cast<double>(h) / static_cast<double>(std::max<int64_t>(nt, 1));
}

// Morton order of the nodes (host; once per mesh): iperm[k] = user id of the k-th node.
void perm_ids_device(const int32_t* perm, const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  k_perm_ids<<<grid_for(n), 256, 0, s>>>(perm, in, out, n);
  FS_LAUNCH_CHECK();
}

__global__ void k_perm_ids_inplace(const int32_t* __restrict__ perm, int32_t* ids, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[k];
    if (v >= 0) ids[k] = perm[v];
  }
}

// ids[k] <- perm[ids[k]] in place (negative ids kept).
void perm_ids_inplace_device(const int32_t* perm, int32_t* ids, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  k_perm_ids_inplace<<<grid_for(n), 256, 0, s>>>(perm, ids, n);
  FS_LAUNCH_CHECK();
}

void perm_ids_valid_device(const int32_t* perm, const int32_t* in, int32_t* out, int64_t n, int64_t nn,
                           cudaStream_t s) {
  if (n <= 0) return;
  k_perm_ids_valid<<<grid_for(n), 256, 0, s>>>(perm, in, out, n, nn);
  FS_LAUNCH_CHECK();
}

void permute_rows_device(const int32_t* iperm, const double* in, double* out, int64_t nn, int w, bool to_internal,
                         cudaStream_t s) {
  if (nn <= 0) return;
  k_permute_rows<double><<<grid_for(nn * w), 256, 0, s>>>(iperm, in, out, nn, w, to_internal);
  FS_LAUNCH_CHECK();
}

void permute_rows_u8_device(const int32_t* iperm, const uint8_t* in, uint8_t* out, int64_t nn, bool to_internal,
                            cudaStream_t s) {
  if (nn <= 0) return;
  k_permute_rows<uint8_t><<<grid_for(nn), 256, 0, s>>>(iperm, in, out, nn, 1, to_internal);
  FS_LAUNCH_CHECK();
}

void export_csr_user_device(const int32_t* perm, const int32_t* iperm, const Pattern& pat, const double* svals,
                            int64_t* uptr /*[nn+1] scratch*/, int64_t* udeg /*[nn+1] scratch*/, void* scan_tmp,
                            size_t scan_tmp_b, int64_t* row_ptr, int32_t* col_idx, double* vals, cudaStream_t s) {
  const int64_t nn = pat.nloc;
  k_user_degrees<<<grid_for(nn), 256, 0, s>>>(perm, pat.node_ptr.get(), nn, udeg);
  FS_LAUNCH_CHECK();
  exclusive_scan_i64(udeg, uptr, nn, s, scan_tmp, scan_tmp_b);
  const int g = static_cast<int>(std::min<int64_t>(ceil_div(nn, kExpWarps), 32LL * num_sms()));
  k_export_csr_user<<<std::max(g, 1), kExpWarps * 32, 0, s>>>(perm, iperm, pat.node_ptr.get(), pat.nbr.get(),
                                                              pat.sptr.get(), pat.sdiag.get(), pat.tptr.get(),
                                                              pat.tlist.get(), svals, uptr, nn, row_ptr, col_idx,
                                                              vals);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
