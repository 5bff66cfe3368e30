// S7 — essential boundary conditions ("removing (or modifying) the rows and
// columns"; "the penalty function method") and the Jacobi preconditioner.
// Clamped nodes only (prescribed displacement g = 0, reading Q8).
#include "common.cuh"

namespace fsfem {

namespace {

__global__ void k_mark_fixed(const int32_t* __restrict__ dir, int64_t nd, int64_t nn, uint8_t* __restrict__ fixed,
                             unsigned long long* __restrict__ err) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nd; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = dir[k];
    if (v < 0 || v >= nn) {
      report_error(err, FSFEM_ERR_INVALID_ARG, k);
      continue;
    }
    fixed[v] = 1;
  }
}

// MODIFY: warp per own node i over its stored blocks (pattern.cuh; the transposed half is the
// same memory).  Block (i, j) is zeroed when i or j is clamped, except the diagonal entries of
// block (i, i).
__global__ void k_bc_modify(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr, int64_t n_lo,
                            int64_t nloc, const uint8_t* __restrict__ fixed, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  for (int64_t il = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; il < nloc;
       il += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t i = static_cast<int32_t>(n_lo + il);
    const bool fi = fixed[i] != 0;
    const int64_t P = node_ptr[il];
    const int deg = static_cast<int>(node_ptr[il + 1] - P);
    double* blocks = vals + 9 * P;
    for (int s = lane; s < deg; s += 32) {
      const int32_t j = nbr[P + s];
      if (!(fi || fixed[j])) continue;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (!(j == i && a == c)) blocks[9 * s + 3 * a + c] = 0.0;
    }
  }
}

// f = loads on own rows; MODIFY also sets f_r = K_rr * g_r = 0 on clamped dofs.
__global__ void k_bc_rhs(const double* __restrict__ loads, const uint8_t* __restrict__ fixed, int64_t n_lo,
                         int64_t nloc, int mode, double* __restrict__ f) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * nloc; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = n_lo + k / 3;
    const double v = loads[3 * n_lo + k];
    f[k] = (mode == 0 && fixed[i]) ? 0.0 : v;
  }
}

// Index of diagonal entry a of own node il, or -1 when the node has no diagonal block (in no tet).
__device__ __forceinline__ int64_t diag_index(const int64_t* node_ptr, const int32_t* diag_slot, int64_t il, int a) {
  const int32_t d = diag_slot[il];
  return d < 0 ? -1 : 9 * (node_ptr[il] + d) + 4 * a;
}

// max_i K_ii over own rows, as the bit pattern of a non-negative double (ordered like integers).
__global__ void k_diag_max(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ diag_slot,
                           const double* __restrict__ vals, int64_t nloc, unsigned long long* __restrict__ out) {
  double mx = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * nloc; k += (int64_t)gridDim.x * blockDim.x)
  {
    const int64_t di = diag_index(node_ptr, diag_slot, k / 3, static_cast<int>(k % 3));
    if (di >= 0) mx = fmax(mx, vals[di]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(mx)));
}

__global__ void k_bc_penalty(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ diag_slot, int64_t n_lo,
                             int64_t nloc, const uint8_t* __restrict__ fixed, const unsigned long long* __restrict__ dmax,
                             double scale, double* __restrict__ vals) {
  const double alpha = scale * __longlong_as_double(static_cast<long long>(*dmax));
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * nloc; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t di = diag_index(node_ptr, diag_slot, k / 3, static_cast<int>(k % 3));
    if (fixed[n_lo + k / 3] && di >= 0) vals[di] += alpha;
  }
}

__global__ void k_dinv(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ diag_slot,
                       const double* __restrict__ vals, int64_t n_lo, int64_t nloc, double* __restrict__ dinv,
                       unsigned long long* __restrict__ err) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3 * nloc; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t di = diag_index(node_ptr, diag_slot, k / 3, static_cast<int>(k % 3));
    const double d = di >= 0 ? vals[di] : 0.0;
    if (!(d > 0.0) || !isfinite(d)) report_error(err, FSFEM_ERR_BREAKDOWN, 3 * n_lo + k);
    dinv[k] = 1.0 / d;
  }
}

}  // namespace

void apply_bc_device(const int64_t* node_ptr, const int32_t* nbr, const int32_t* diag_slot, int64_t n_lo, int64_t nloc,
                     int64_t nn, const int32_t* dir, int64_t nd, const double* loads, int mode, double penalty_scale,
                     double* vals, double* f, double* dinv, uint8_t* fixed, unsigned long long* flags /*[2]*/,
                     cudaStream_t s) {
  const int sms = num_sms();
  FS_CUDA(cudaMemsetAsync(fixed, 0, nn, s));
  FS_CUDA(cudaMemsetAsync(flags, 0xff, sizeof(unsigned long long), s));
  FS_CUDA(cudaMemsetAsync(flags + 1, 0, sizeof(unsigned long long), s));
  if (nd > 0) {
    k_mark_fixed<<<static_cast<int>(std::min<int64_t>(ceil_div(nd, 256), 4LL * sms)), 256, 0, s>>>(dir, nd, nn, fixed,
                                                                                                   flags);
    FS_LAUNCH_CHECK();
  }
  const int gv = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(3 * nloc, 256), 8LL * sms)));
  const int gw = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(32 * nloc, 256), 32LL * sms)));
  if (mode == 0) {
    k_bc_modify<<<gw, 256, 0, s>>>(node_ptr, nbr, n_lo, nloc, fixed, vals);
    FS_LAUNCH_CHECK();
  } else {
    k_diag_max<<<gv, 256, 0, s>>>(node_ptr, diag_slot, vals, nloc, flags + 1);
    FS_LAUNCH_CHECK();
    k_bc_penalty<<<gv, 256, 0, s>>>(node_ptr, diag_slot, n_lo, nloc, fixed, flags + 1,
                                    penalty_scale > 0.0 ? penalty_scale : 1e8, vals);
    FS_LAUNCH_CHECK();
  }
  k_bc_rhs<<<gv, 256, 0, s>>>(loads, fixed, n_lo, nloc, mode, f);
  FS_LAUNCH_CHECK();
  k_dinv<<<gv, 256, 0, s>>>(node_ptr, diag_slot, vals, n_lo, nloc, dinv, flags);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
