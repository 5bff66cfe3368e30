// Deterministic exclusive prefix sums (reduce -> scan of tile sums -> scan with offsets).
// Used for bucket offsets (S1), incidence / pattern pointers (S5).  Integer-only, so the
// result is exact and independent of the launch shape.
#include "common.cuh"

namespace fsfem {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total via *total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T w = (lane < kScanThreads / 32) ? warp_tot[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < kScanThreads / 32) warp_tot[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  T r = inc - v + warp_tot[wid];
  __syncthreads();
  return r;
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kScanThreads) k_tile_reduce(const Tin* __restrict__ in, int64_t n,
                                                              Tout* __restrict__ sums) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  Tout s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + static_cast<int64_t>(k) * kScanThreads + threadIdx.x;
    if (i < n) s += static_cast<Tout>(in[i]);
  }
  __shared__ Tout tot;
  block_excl_scan<Tout>(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// One block scans the tile sums (exclusive), serially in chunks of kScanThreads.
template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(T* sums, int64_t nb) {
  __shared__ T carry_s;
  __shared__ T tot;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
    const int64_t i = b0 + threadIdx.x;
    T v = (i < nb) ? sums[i] : T(0);
    T e = block_excl_scan<T>(v, &tot);
    const T carry = carry_s;
    if (i < nb) sums[i] = e + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = carry_s;
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const Tin* __restrict__ in, Tout* __restrict__ out,
                                                            int64_t n, const Tout* __restrict__ sums) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  // each thread owns kScanItems consecutive items
  Tout v[kScanItems];
  Tout s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + static_cast<int64_t>(threadIdx.x) * kScanItems + k;
    v[k] = (i < n) ? static_cast<Tout>(in[i]) : Tout(0);
    s += v[k];
  }
  __shared__ Tout tot;
  Tout e = block_excl_scan<Tout>(s, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + static_cast<int64_t>(threadIdx.x) * kScanItems + k;
    if (i < n) out[i] = e;
    e += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = sums[gridDim.x];
}

template <typename Tin, typename Tout>
void scan_impl(const Tin* in, Tout* out, int64_t n, cudaStream_t s, void* tmp, size_t tmp_bytes) {
  if (n <= 0) {
    FS_CUDA(cudaMemsetAsync(out, 0, sizeof(Tout), s));
    return;
  }
  const int64_t nb = ceil_div(n, kTile);
  if (tmp_bytes < sizeof(Tout) * static_cast<size_t>(nb + 1)) throw Error(FSFEM_ERR_CUDA, "scan: temp too small");
  Tout* sums = static_cast<Tout*>(tmp);
  k_tile_reduce<Tin, Tout><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, sums);
  FS_LAUNCH_CHECK();
  k_scan_sums<Tout><<<1, kScanThreads, 0, s>>>(sums, nb);
  FS_LAUNCH_CHECK();
  k_tile_scan<Tin, Tout><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, out, n, sums);
  FS_LAUNCH_CHECK();
}

}  // namespace

size_t scan_tmp_bytes(int64_t n) { return sizeof(int64_t) * static_cast<size_t>(ceil_div(n, kTile) + 2); }

void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s, void* tmp, size_t tb) {
  scan_impl<int32_t, int32_t>(in, out, n, s, tmp, tb);
}
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s, void* tmp, size_t tb) {
  scan_impl<int64_t, int64_t>(in, out, n, s, tmp, tb);
}
void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s, void* tmp, size_t tb) {
  scan_impl<int32_t, int64_t>(in, out, n, s, tmp, tb);
}

}  // namespace fsfem
