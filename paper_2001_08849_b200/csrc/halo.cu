// Halo-only exchange of the search direction for the row partition.
//
// Rank r owns nodes [n_lo, n_hi) and stores rows that reference other ranks' nodes only through
// the columns of its rows (symmetric storage: stored blocks j >= i plus halo blocks j < n_lo; the
// transposed blocks are rank-local).  The halo of rank r is the set of those columns outside its
// range: before each SpMV only these entries of p are needed from the other ranks, instead of
// the whole vector (the all-gather).  Here: the halo list (global node ids, ascending, hence
// grouped by owner rank) and the pack / unpack kernels; the exchange itself is NCCL send/recv
// in api.cu.
#include "common.cuh"
#include <algorithm>
#include <vector>
#include "pattern.cuh"

namespace fsfem {

namespace {

__global__ void k_halo_mark(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr, int64_t nloc,
                            int64_t n_lo, int64_t n_hi, int32_t* __restrict__ flag) {
  const int64_t nb = node_ptr[nloc];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nb; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = nbr[k];
    if (j < n_lo || j >= n_hi) flag[j] = 1;  // same value from every writer
  }
}

__global__ void k_halo_compact(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos, int64_t nn,
                               int32_t* __restrict__ halo) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nn; j += (int64_t)gridDim.x * blockDim.x)
    if (flag[j]) halo[pos[j]] = static_cast<int32_t>(j);
}

__global__ void k_halo_pack(const double* __restrict__ full, const int32_t* __restrict__ nodes, int64_t n,
                            double* __restrict__ buf) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * n; k += (int64_t)gridDim.x * blockDim.x)
    buf[k] = full[3 * static_cast<int64_t>(nodes[k / 3]) + k % 3];
}

__global__ void k_halo_unpack(const double* __restrict__ buf, const int32_t* __restrict__ nodes, int64_t n,
                              double* __restrict__ full) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * n; k += (int64_t)gridDim.x * blockDim.x)
    full[3 * static_cast<int64_t>(nodes[k / 3]) + k % 3] = buf[k];
}

int grid_n(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 8LL * num_sms())));
}

}  // namespace

// Halo list of the rank (pat.halo, ascending global ids) and its size; per-owner counts on the
// host (owner q holds nodes [ranges[q], ranges[q + 1])).
void build_halo_device(Pattern& pat, int64_t nn, const std::vector<int64_t>& ranges, std::vector<int64_t>& need,
                       DevBuf<unsigned char>& scratch, cudaStream_t s) {
  const int nranks = static_cast<int>(ranges.size()) - 1;
  const int64_t n_hi = pat.n_lo + pat.nloc;
  const size_t tb = scan_tmp_bytes(nn + 1);
  const size_t o_flag = 0, o_pos = (sizeof(int32_t) * (nn + 1) + 255) & ~size_t(255),
               o_tmp = o_pos + ((sizeof(int32_t) * (nn + 1) + 255) & ~size_t(255));
  unsigned char* b = scratch.ensure(o_tmp + tb);
  int32_t* flag = reinterpret_cast<int32_t*>(b + o_flag);
  int32_t* pos = reinterpret_cast<int32_t*>(b + o_pos);
  FS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t) * (nn + 1), s));
  if (pat.nloc > 0) {
    k_halo_mark<<<grid_n(pat.nblk), 256, 0, s>>>(pat.node_ptr.get(), pat.nbr.get(), pat.nloc, pat.n_lo, n_hi, flag);
    FS_LAUNCH_CHECK();
  }
  exclusive_scan_i32(flag, pos, nn, s, b + o_tmp, tb);
  int32_t nh = 0;
  FS_CUDA(cudaMemcpyAsync(&nh, pos + nn, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  pat.nhalo = nh;
  pat.halo.ensure(std::max<int64_t>(nh, 1));
  k_halo_compact<<<grid_n(nn), 256, 0, s>>>(flag, pos, nn, pat.halo.get());
  FS_LAUNCH_CHECK();
  std::vector<int32_t> h(nh);
  if (nh > 0) FS_CUDA(cudaMemcpyAsync(h.data(), pat.halo.get(), sizeof(int32_t) * nh, cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  need.assign(nranks, 0);
  for (int32_t j : h) {
    const int q = static_cast<int>(std::upper_bound(ranges.begin(), ranges.end(), static_cast<int64_t>(j)) -
                                   ranges.begin()) - 1;
    need[std::min(nranks - 1, std::max(0, q))] += 1;
  }
}

void halo_pack_device(const double* full, const int32_t* nodes, int64_t n, double* buf, cudaStream_t s) {
  if (n <= 0) return;
  k_halo_pack<<<grid_n(3 * n), 256, 0, s>>>(full, nodes, n, buf);
  FS_LAUNCH_CHECK();
}

void halo_unpack_device(const double* buf, const int32_t* nodes, int64_t n, double* full, cudaStream_t s) {
  if (n <= 0) return;
  k_halo_unpack<<<grid_n(3 * n), 256, 0, s>>>(buf, nodes, n, full);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
