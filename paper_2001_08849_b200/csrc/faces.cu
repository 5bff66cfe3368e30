// S1 — face extraction (Fig. 7, Alg. 1), re-designed for the GPU.
//
// The paper looks up, for every row of TetGen's face file, the tet(s) that own it
// (Alg. 1, a data-parallel loop with SharedArrays).  Here faces are derived from the tets
// alone by an MSD radix sort on the packed sorted-vertex key (a, b, c):
//   1. digit = a = smallest vertex of the face (radix N_n): counting sort of the 4*N_t face
//      instances into per-node buckets (histogram + exclusive scan + scatter);
//   2. inside each bucket (<= ~72 instances on the paper-like meshes) a warp sorts the
//      remaining key (b, c) together with the payload 4t+l in shared memory;
//   3. equal keys form runs of length 1 (exterior face) or 2 (interior face, t0 < t1
//      because the payload breaks ties); length > 2 is a TOPOLOGY error.
// The output order is ascending (a, b, c), the same total order as the oracle's map.
#include "common.cuh"

namespace fsfem {

namespace {

constexpr int kSortWarps = 4;     // warps per CTA in the bucket kernels (24 KB smem)
constexpr int kBucketCap = 256;   // instances a warp sorts in shared memory
constexpr int kBigCap = 4096;     // instances a CTA sorts in shared memory (rare buckets)

__device__ __forceinline__ void face_of(const int4 v, int l, int& a, int& b, int& c) {
  // the face opposite local vertex l, vertices sorted ascending
  int x, y, z;
  if (l == 0) { x = v.y; y = v.z; z = v.w; }
  else if (l == 1) { x = v.x; y = v.z; z = v.w; }
  else if (l == 2) { x = v.x; y = v.y; z = v.w; }
  else { x = v.x; y = v.y; z = v.z; }
  a = min(x, min(y, z));
  c = max(x, max(y, z));
  b = x + y + z - a - c;
}

// Partial bounding boxes: block b writes (min x, min y, min z, max x, max y, max z).
__global__ void k_bbox_partial(const double* __restrict__ xyz, int64_t nn, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double x = xyz[3 * i + a];
      lo[a] = fmin(lo[a], x);
      hi[a] = fmax(hi[a], x);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  __shared__ double s[32][6];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) { s[wid][a] = lo[a]; s[wid][3 + a] = hi[a]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    double r = s[0][threadIdx.x];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      r = threadIdx.x < 3 ? fmin(r, s[w][threadIdx.x]) : fmax(r, s[w][threadIdx.x]);
    part[6 * blockIdx.x + threadIdx.x] = r;
  }
}

// One block of 256 threads: strided partial reductions, then warp trees (min/max are exact and
// order-independent).
__global__ void __launch_bounds__(256) k_bbox_final(const double* __restrict__ part, int nparts,
                                                    double* __restrict__ bbox) {
  double r[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < nparts; b += blockDim.x)
#pragma unroll
    for (int a = 0; a < 6; ++a) r[a] = a < 3 ? fmin(r[a], part[6 * b + a]) : fmax(r[a], part[6 * b + a]);
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v = __shfl_xor_sync(0xffffffffu, r[a], o);
      r[a] = a < 3 ? fmin(r[a], v) : fmax(r[a], v);
    }
  __shared__ double s[8][6];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int a = 0; a < 6; ++a) s[wid][a] = r[a];
  __syncthreads();
  if (threadIdx.x < 6) {
    double v = s[0][threadIdx.x];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      v = threadIdx.x < 3 ? fmin(v, s[w][threadIdx.x]) : fmax(v, s[w][threadIdx.x]);
    bbox[threadIdx.x] = v;
  }
}

// Validate each tet (ids, repeated nodes, |V_e| threshold) and histogram its 4 faces by
// their smallest vertex.
__global__ void k_face_count(const int4* __restrict__ tets, int64_t nt, int64_t nn, const double* __restrict__ xyz,
                             const double* __restrict__ bbox, int32_t* __restrict__ cnt,
                             unsigned long long* __restrict__ err) {
  const double dx = bbox[3] - bbox[0], dy = bbox[4] - bbox[1], dz = bbox[5] - bbox[2];
  const double diag = sqrt(dx * dx + dy * dy + dz * dz);
  const double tol = 1e-14 * diag * diag * diag;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = tets[t];
    if (v.x < 0 || v.y < 0 || v.z < 0 || v.w < 0 || v.x >= nn || v.y >= nn || v.z >= nn || v.w >= nn) {
      report_error(err, FSFEM_ERR_INVALID_ARG, t);
      continue;
    }
    if (v.x == v.y || v.x == v.z || v.x == v.w || v.y == v.z || v.y == v.w || v.z == v.w) {
      report_error(err, FSFEM_ERR_DEGENERATE, t);
      continue;
    }
    const double x0 = xyz[3 * v.x], y0 = xyz[3 * v.x + 1], z0 = xyz[3 * v.x + 2];
    const double e1x = xyz[3 * v.y] - x0, e1y = xyz[3 * v.y + 1] - y0, e1z = xyz[3 * v.y + 2] - z0;
    const double e2x = xyz[3 * v.z] - x0, e2y = xyz[3 * v.z + 1] - y0, e2z = xyz[3 * v.z + 2] - z0;
    const double e3x = xyz[3 * v.w] - x0, e3y = xyz[3 * v.w + 1] - y0, e3z = xyz[3 * v.w + 2] - z0;
    const double det = e1x * (e2y * e3z - e2z * e3y) - e1y * (e2x * e3z - e2z * e3x) + e1z * (e2x * e3y - e2y * e3x);
    if (!(fabs(det) / 6.0 > tol)) report_error(err, FSFEM_ERR_DEGENERATE, t);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      int a, b, c;
      face_of(v, l, a, b, c);
      atomicAdd(&cnt[a], 1);
    }
  }
}

// Scatter each face instance into its bucket: key = (b << 32) | c, payload = 4t + l.
// The slot inside a bucket is arbitrary (atomic cursor); the in-bucket sort fixes the order.
// Tets the count kernel skipped (ids out of range, repeated nodes) are skipped here too, so the
// bucket offsets stay consistent and the build can run to its end before the host looks at errors.
__global__ void k_face_scatter(const int4* __restrict__ tets, int64_t nt, int64_t nn, const int32_t* __restrict__ off,
                               int32_t* __restrict__ cursor, unsigned long long* __restrict__ keys,
                               uint32_t* __restrict__ pay) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = tets[t];
    if (v.x < 0 || v.y < 0 || v.z < 0 || v.w < 0 || v.x >= nn || v.y >= nn || v.z >= nn || v.w >= nn) continue;
    if (v.x == v.y || v.x == v.z || v.x == v.w || v.y == v.z || v.y == v.w || v.z == v.w) continue;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      int a, b, c;
      face_of(v, l, a, b, c);
      const int32_t pos = off[a] + atomicAdd(&cursor[a], 1);
      keys[pos] = (static_cast<unsigned long long>(b) << 32) | static_cast<uint32_t>(c);
      pay[pos] = static_cast<uint32_t>(4 * t + l);
    }
  }
}

__device__ __forceinline__ bool key_less(unsigned long long ka, uint32_t pa, unsigned long long kb, uint32_t pb) {
  return ka < kb || (ka == kb && pa < pb);
}

// Sort one bucket staged in shared memory (sk/sp, n items) into ok/op by rank
// (rank = number of strictly smaller (key, payload) pairs; all pairs are distinct).
// `t0`/`nthr` = this thread's index / the number of cooperating threads.
__device__ __forceinline__ void rank_sort(const unsigned long long* sk, const uint32_t* sp,
                                          unsigned long long* ok, uint32_t* op, int n, int t0, int nthr) {
  for (int i = t0; i < n; i += nthr) {
    const unsigned long long ki = sk[i];
    const uint32_t pi = sp[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += key_less(sk[j], sp[j], ki, pi) ? 1 : 0;
    ok[r] = ki;
    op[r] = pi;
  }
}

template <int kThreads>
__device__ __forceinline__ void finish_bucket(const unsigned long long* ok, const uint32_t* op, int n, int t0,
                                              unsigned long long* __restrict__ keys, uint32_t* __restrict__ pay,
                                              int32_t beg, int& starts, bool& too_long) {
  for (int i = t0; i < n; i += kThreads) {
    const unsigned long long k = ok[i];
    keys[beg + i] = k;
    pay[beg + i] = op[i];
    if (i == 0 || ok[i - 1] != k) ++starts;
    if (i >= 2 && ok[i - 2] == k) too_long = true;
  }
}

// Warp per bucket (node a).  Buckets larger than kBucketCap are deferred to k_bucket_sort_big.
__global__ void __launch_bounds__(kSortWarps * 32) k_bucket_sort(const int32_t* __restrict__ off, int64_t nn,
                                                                 unsigned long long* __restrict__ keys,
                                                                 uint32_t* __restrict__ pay, int32_t* __restrict__ ucnt,
                                                                 int32_t* __restrict__ big_list, int32_t* __restrict__ n_big,
                                                                 unsigned long long* __restrict__ err) {
  __shared__ unsigned long long sk[kSortWarps][kBucketCap], ok[kSortWarps][kBucketCap];
  __shared__ uint32_t sp[kSortWarps][kBucketCap], op[kSortWarps][kBucketCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kSortWarps;
  for (int64_t a = blockIdx.x * (int64_t)kSortWarps + w; a < nn; a += nwarps) {
    const int32_t beg = off[a];
    const int n = off[a + 1] - beg;
    if (n > kBucketCap) {
      if (lane == 0) {
        big_list[atomicAdd(n_big, 1)] = static_cast<int32_t>(a);
        ucnt[a] = 0;
      }
      continue;
    }
    if (n <= 32) {  // one instance per lane: bitonic network on (key, payload) in registers
      unsigned long long k = lane < n ? keys[beg + lane] : ~0ull;
      uint32_t p = lane < n ? pay[beg + lane] : 0xffffffffu;
#pragma unroll
      for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
          const unsigned long long ko = __shfl_xor_sync(0xffffffffu, k, j);
          const uint32_t po = __shfl_xor_sync(0xffffffffu, p, j);
          const bool keep_min = ((lane & j) == 0) == ((lane & size) == 0);
          const bool other_less = key_less(ko, po, k, p);
          if (keep_min ? other_less : !other_less) {
            k = ko;
            p = po;
          }
        }
      }
      if (lane < n) {
        keys[beg + lane] = k;
        pay[beg + lane] = p;
      }
      const unsigned long long k1 = __shfl_up_sync(0xffffffffu, k, 1), k2 = __shfl_up_sync(0xffffffffu, k, 2);
      const bool start = lane < n && (lane == 0 || k1 != k);
      const bool too_long = lane < n && lane >= 2 && k2 == k;
      const int starts = __popc(__ballot_sync(0xffffffffu, start));
      if (__any_sync(0xffffffffu, too_long) && lane == 0) report_error(err, FSFEM_ERR_TOPOLOGY, a);
      if (lane == 0) ucnt[a] = starts;
      continue;
    }
    for (int i = lane; i < n; i += 32) {
      sk[w][i] = keys[beg + i];
      sp[w][i] = pay[beg + i];
    }
    __syncwarp();
    bool too_long = false;
    rank_sort(sk[w], sp[w], ok[w], op[w], n, lane, 32);
    __syncwarp();
    int starts = 0;
    finish_bucket<32>(ok[w], op[w], n, lane, keys, pay, beg, starts, too_long);
    starts = __reduce_add_sync(0xffffffffu, starts);
    if (__any_sync(0xffffffffu, too_long) && lane == 0) report_error(err, FSFEM_ERR_TOPOLOGY, a);
    if (lane == 0) ucnt[a] = starts;
    __syncwarp();
  }
}

// CTA per large bucket (dynamic shared memory, up to kBigCap instances).
__global__ void __launch_bounds__(256) k_bucket_sort_big(const int32_t* __restrict__ off, const int32_t* __restrict__ big_list,
                                                         const int32_t* __restrict__ n_big,
                                                         unsigned long long* __restrict__ keys, uint32_t* __restrict__ pay,
                                                         int32_t* __restrict__ ucnt, unsigned long long* __restrict__ err) {
  extern __shared__ unsigned long long dyn[];
  const int nb = *n_big;  // written by k_bucket_sort (no host round trip)
  for (int ib = blockIdx.x; ib < nb; ib += gridDim.x) {
  const int32_t a = big_list[ib];
  const int32_t beg = off[a];
  const int n = off[a + 1] - beg;
  if (n > kBigCap) {
    if (threadIdx.x == 0) report_error(err, FSFEM_ERR_UNSUPPORTED, a);
    continue;  // uniform over the CTA
  }
  unsigned long long* sk = dyn;
  unsigned long long* ok = sk + kBigCap;
  uint32_t* sp = reinterpret_cast<uint32_t*>(ok + kBigCap);
  uint32_t* op = sp + kBigCap;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sk[i] = keys[beg + i];
    sp[i] = pay[beg + i];
  }
  __syncthreads();
  bool too_long = false;
  rank_sort(sk, sp, ok, op, n, threadIdx.x, blockDim.x);
  __syncthreads();
  int starts = 0;
  finish_bucket<256>(ok, op, n, threadIdx.x, keys, pay, beg, starts, too_long);
  __shared__ int tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  atomicAdd(&tot, starts);
  if (too_long) report_error(err, FSFEM_ERR_TOPOLOGY, a);
  __syncthreads();
  if (threadIdx.x == 0) ucnt[a] = tot;
  __syncthreads();  // sk / ok / tot are reused by the next bucket
  }
}

// Warp per bucket: emit the faces of bucket a at face ids foff[a] + run index.
__global__ void __launch_bounds__(256) k_face_emit(const int32_t* __restrict__ off, const int32_t* __restrict__ foff,
                                                   int64_t nn, const unsigned long long* __restrict__ keys,
                                                   const uint32_t* __restrict__ pay, const int32_t* __restrict__ tets,
                                                   int32_t* __restrict__ face_nodes, int32_t* __restrict__ face_tet,
                                                   int32_t* __restrict__ face_opp, int32_t* __restrict__ tet_face,
                                                   int32_t* __restrict__ tet_across,
                                                   unsigned long long* __restrict__ n_interior) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned int interior = 0;
  for (int64_t a = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); a < nn; a += nwarps) {
    const int32_t beg = off[a];
    const int n = off[a + 1] - beg;
    int32_t fid_base = foff[a] - 1;  // id of the run containing the current element
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int i = c0 + lane;
      const bool valid = i < n;
      unsigned long long k = 0, kprev = 0, knext = ~0ull;
      uint32_t p = 0, pnext = 0;
      if (valid) {
        k = keys[beg + i];
        p = pay[beg + i];
        if (i > 0) kprev = keys[beg + i - 1];
        if (i + 1 < n) {
          knext = keys[beg + i + 1];
          pnext = pay[beg + i + 1];
        }
      }
      const bool start = valid && (i == 0 || kprev != k);
      const unsigned int ball = __ballot_sync(0xffffffffu, start);
      const int32_t fid = fid_base + __popc(ball & ((2u << lane) - 1u));
      if (valid) {
        tet_face[p] = fid;
        if (start) {
          const int32_t t0 = static_cast<int32_t>(p >> 2);
          face_nodes[3 * fid] = static_cast<int32_t>(a);
          face_nodes[3 * fid + 1] = static_cast<int32_t>(k >> 32);
          face_nodes[3 * fid + 2] = static_cast<int32_t>(k & 0xffffffffu);
          face_tet[2 * fid] = t0;
          face_opp[2 * fid] = tets[p];  // tets[4*t0 + l] with p = 4*t0 + l
          if (knext == k) {
            face_tet[2 * fid + 1] = static_cast<int32_t>(pnext >> 2);
            face_opp[2 * fid + 1] = tets[pnext];
            tet_across[p] = tets[pnext];  // the vertex across face l of tet t, seen from each side
            tet_across[pnext] = tets[p];
            ++interior;
          } else {
            face_tet[2 * fid + 1] = -1;
            face_opp[2 * fid + 1] = -1;
            tet_across[p] = -1;
          }
        }
      }
      fid_base += __popc(ball);
    }
  }
  interior = __reduce_add_sync(0xffffffffu, interior);
  if (lane == 0 && interior) atomicAdd(n_interior, static_cast<unsigned long long>(interior));
}

}  // namespace

// Host driver of S1.  All device buffers belong to the context.
void build_faces_device(const double* d_xyz, int64_t nn, const int32_t* d_tets, int64_t nt, cudaStream_t s,
                        DevBuf<unsigned char>& scratch, DevBuf<int32_t>& face_nodes, DevBuf<int32_t>& face_tet,
                        DevBuf<int32_t>& face_opp, DevBuf<int32_t>& tet_face, DevBuf<int32_t>& tet_across,
                        int64_t* n_faces, int64_t* n_interior, unsigned long long* h_flags /* pinned [4] */) {
  const int64_t nk = 4 * nt;
  const int sms = num_sms();
  // scratch layout
  size_t o = 0;
  auto carve = [&](size_t bytes) {
    size_t at = o;
    o += (bytes + 255) & ~size_t(255);
    return at;
  };
  const size_t o_cnt = carve(sizeof(int32_t) * (nn + 1));
  const size_t o_off = carve(sizeof(int32_t) * (nn + 1));
  const size_t o_cur = carve(sizeof(int32_t) * (nn + 1));
  const size_t o_ucnt = carve(sizeof(int32_t) * (nn + 1));
  const size_t o_foff = carve(sizeof(int32_t) * (nn + 1));
  const size_t o_keys = carve(sizeof(unsigned long long) * nk);
  const size_t o_pay = carve(sizeof(uint32_t) * nk);
  const size_t o_big = carve(sizeof(int32_t) * (nn + 1));
  const size_t o_bbp = carve(sizeof(double) * 6 * 1024);
  const size_t o_bb = carve(sizeof(double) * 8);
  const size_t o_flags = carve(sizeof(unsigned long long) * 4);
  const size_t o_tmp = carve(scan_tmp_bytes(nn + 1));
  unsigned char* base = scratch.ensure(o);
  auto at = [&](size_t off) { return static_cast<void*>(base + off); };
  int32_t* cnt = static_cast<int32_t*>(at(o_cnt));
  int32_t* off = static_cast<int32_t*>(at(o_off));
  int32_t* cur = static_cast<int32_t*>(at(o_cur));
  int32_t* ucnt = static_cast<int32_t*>(at(o_ucnt));
  int32_t* foff = static_cast<int32_t*>(at(o_foff));
  unsigned long long* keys = static_cast<unsigned long long*>(at(o_keys));
  uint32_t* pay = static_cast<uint32_t*>(at(o_pay));
  int32_t* big = static_cast<int32_t*>(at(o_big));
  double* bbp = static_cast<double*>(at(o_bbp));
  double* bb = static_cast<double*>(at(o_bb));
  unsigned long long* flags = static_cast<unsigned long long*>(at(o_flags));
  void* tmp = at(o_tmp);
  const size_t tmp_bytes = scan_tmp_bytes(nn + 1);

  FS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nn + 1), s));
  FS_CUDA(cudaMemsetAsync(cur, 0, sizeof(int32_t) * (nn + 1), s));
  FS_CUDA(cudaMemsetAsync(flags, 0xff, sizeof(unsigned long long), s));      // [0] validation errors
  FS_CUDA(cudaMemsetAsync(flags + 1, 0, sizeof(unsigned long long) * 2, s));  // [1] interior, [2] big buckets
  FS_CUDA(cudaMemsetAsync(flags + 3, 0xff, sizeof(unsigned long long), s));  // [3] sort errors
  PhaseTimer pt(s, "faces");

  // One host round trip for the whole build: invalid tets are skipped by count and scatter alike,
  // big buckets are found on the device, and the outputs are sized by the bound N_f <= 4 N_t.
  const int nbb = static_cast<int>(std::min<int64_t>(1024, std::max<int64_t>(1, ceil_div(nn, 256))));
  k_bbox_partial<<<nbb, 256, 0, s>>>(d_xyz, nn, bbp);
  FS_LAUNCH_CHECK();
  k_bbox_final<<<1, 256, 0, s>>>(bbp, nbb, bb);
  FS_LAUNCH_CHECK();
  const int grid_t = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nt, 256), 8LL * sms)));
  k_face_count<<<grid_t, 256, 0, s>>>(reinterpret_cast<const int4*>(d_tets), nt, nn, d_xyz, bb, cnt, flags);
  FS_LAUNCH_CHECK();
  exclusive_scan_i32(cnt, off, nn, s, tmp, tmp_bytes);
  k_face_scatter<<<grid_t, 256, 0, s>>>(reinterpret_cast<const int4*>(d_tets), nt, nn, off, cur, keys, pay);
  FS_LAUNCH_CHECK();
  const int grid_b = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nn, kSortWarps), 16LL * sms)));
  k_bucket_sort<<<grid_b, kSortWarps * 32, 0, s>>>(off, nn, keys, pay, ucnt, big,
                                                   reinterpret_cast<int32_t*>(flags + 2), flags + 3);
  FS_LAUNCH_CHECK();
  {
    const size_t smem = (2 * sizeof(unsigned long long) + 2 * sizeof(uint32_t)) * kBigCap;
    static bool attr = false;
    if (!attr) {
      FS_CUDA(cudaFuncSetAttribute(k_bucket_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    k_bucket_sort_big<<<sms, 256, smem, s>>>(off, big, reinterpret_cast<const int32_t*>(flags + 2), keys, pay, ucnt,
                                             flags + 3);
    FS_LAUNCH_CHECK();
  }
  exclusive_scan_i32(ucnt, foff, nn, s, tmp, tmp_bytes);
  face_nodes.ensure(3 * 4 * nt);
  face_tet.ensure(2 * 4 * nt);
  face_opp.ensure(2 * 4 * nt);
  tet_face.ensure(4 * nt);
  tet_across.ensure(4 * nt);
  k_face_emit<<<grid_b, 256, 0, s>>>(off, foff, nn, keys, pay, d_tets, face_nodes.get(), face_tet.get(),
                                     face_opp.get(), tet_face.get(), tet_across.get(), flags + 1);
  FS_LAUNCH_CHECK();
  int32_t nf32 = 0;
  FS_CUDA(cudaMemcpyAsync(h_flags, flags, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaMemcpyAsync(&nf32, foff + nn, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  pt.mark("faces (one round trip)");
  if (h_flags[0] == kNoError) h_flags[0] = h_flags[3];  // validation errors first (as before)
  if (h_flags[0] != kNoError) return;  // caller decodes
  *n_faces = nf32;
  *n_interior = static_cast<int64_t>(h_flags[1]);
}

// Coordinate bounding box (lo xyz, hi xyz) into bbox[6] on the device (min/max: exact, any order).
void bbox_device(const double* d_xyz, int64_t nn, double* part /*[6 * 16 * num_sms]*/, double* bbox, cudaStream_t s) {
  const int nbb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nn, 256), 16LL * num_sms())));
  k_bbox_partial<<<nbb, 256, 0, s>>>(d_xyz, nn, part);
  FS_LAUNCH_CHECK();
  k_bbox_final<<<1, 256, 0, s>>>(part, nbb, bbox);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
