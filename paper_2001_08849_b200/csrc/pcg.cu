// S8-S9 — Jacobi-preconditioned CG on the assembled CSR (the paper solves with PARDISO,
// PAPER.md:365/449; the north star replaces it by PCG, reading Q9):
//   r = f - K x0, z = D^-1 r, p = z, rho = r.z
//   loop: q = K p; alpha = rho / p.q; x += alpha p; r -= alpha q;
//         stop if ||r|| <= tol ||f||; z = D^-1 r; rho' = r.z; beta = rho'/rho; p = z + beta p
// Three kernels per iteration (SpMV+dot, update+dots, direction).  Every dot product is a
// fixed-shape tree (warp shuffles, fixed CTA order, "last CTA reduces") so results are
// bitwise reproducible.  Scalars live on the device; the host only polls `done` between
// CUDA-graph batches of iterations.
#include "common.cuh"
#include "pcg.cuh"

namespace fsfem {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// Deterministic CTA sum of one double per thread (result valid in thread 0).
__device__ __forceinline__ double block_sum(double v, double* sh /*[kWarps]*/) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < kWarps; ++k) r += sh[k];
  __syncthreads();
  return r;
}

// "Last CTA done" pattern: every CTA publishes NV partial sums; the CTA that arrives last sums
// all partials in a fixed tree and returns true (results in out[0..NV) of thread 0).
template <int NV>
__device__ __forceinline__ bool grid_reduce(const double (&mine)[NV], double* part, unsigned int* ticket, double* out) {
  __shared__ double sh[kWarps];
  __shared__ bool last;
  double tot[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) tot[v] = block_sum(mine[v], sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v) part[v * gridDim.x + blockIdx.x] = tot[v];
    __threadfence();
    last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += kThreads) s += ld_cg(part + v * gridDim.x + b);
    out[v] = block_sum(s, sh);
  }
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// Warp per own node: y[3il + a] = sum_k vals[9P + a*3deg + k] * x[3*nbr[P + k/3] + k%3].
// Returns (in lane 0) the three row sums.
__device__ __forceinline__ void node_rows(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr,
                                          const double* __restrict__ vals, const double* __restrict__ x, int64_t il,
                                          double& y0, double& y1, double& y2) {
  const int lane = threadIdx.x & 31;
  const int64_t P = node_ptr[il];
  const int m = static_cast<int>(3 * (node_ptr[il + 1] - P));
  const double* __restrict__ r0 = vals + 9 * P;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int k = lane; k < m; k += 32) {
    const int jb = k / 3;
    const double xv = __ldg(x + 3 * static_cast<int64_t>(__ldg(nbr + P + jb)) + (k - 3 * jb));
    s0 = fma(__ldcs(r0 + k), xv, s0);
    s1 = fma(__ldcs(r0 + m + k), xv, s1);
    s2 = fma(__ldcs(r0 + 2 * m + k), xv, s2);
  }
  y0 = warp_sum(s0);
  y1 = warp_sum(s1);
  y2 = warp_sum(s2);
}

// q = K p on own rows (+ partial p.q, reduced by the last CTA into alpha).
template <bool kPcg>
__global__ void __launch_bounds__(kThreads) k_spmv(const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ nbr,
                                                   const double* __restrict__ vals, int64_t nloc,
                                                   const double* __restrict__ x_full, int64_t own_off,
                                                   double* __restrict__ y, PcgState* st, double* part) {
  if (kPcg && ld_cg(&st->done_d) != 0.0) return;
  const int lane = threadIdx.x & 31;
  double dot = 0.0;
  for (int64_t il = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; il < nloc;
       il += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double y0, y1, y2;
    node_rows(node_ptr, nbr, vals, x_full, il, y0, y1, y2);
    if (lane == 0) {
      y[3 * il] = y0;
      y[3 * il + 1] = y1;
      y[3 * il + 2] = y2;
      if (kPcg) {
        const double* xo = x_full + own_off + 3 * il;
        dot = fma(xo[0], y0, dot);
        dot = fma(xo[1], y1, dot);
        dot = fma(xo[2], y2, dot);
      }
    }
  }
  if (!kPcg) return;
  const double mine[1] = {dot};
  double out[1];
  if (grid_reduce<1>(mine, part, &st->ticket[0], out) && threadIdx.x == 0) {
    if (st->nranks > 1) {
      st->local[0] = out[0];  // combined across ranks by the host-side collective
    } else {
      finish_alpha(st, out[0]);
    }
  }
}

// x += alpha p; r -= alpha q; partial r.r and r.z with z = dinv r.
__global__ void __launch_bounds__(kThreads) k_update(double* __restrict__ x, double* __restrict__ r,
                                                     const double* __restrict__ p, const double* __restrict__ q,
                                                     const double* __restrict__ dinv, int64_t n, PcgState* st,
                                                     double* part) {
  if (ld_cg(&st->done_d) != 0.0) return;
  const double alpha = ld_cg(&st->alpha);
  double rr = 0.0, rz = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    x[k] = fma(alpha, p[k], x[k]);
    const double rk = fma(-alpha, q[k], r[k]);
    r[k] = rk;
    rr = fma(rk, rk, rr);
    rz = fma(rk, dinv[k] * rk, rz);
  }
  const double mine[2] = {rr, rz};
  double out[2];
  if (grid_reduce<2>(mine, part, &st->ticket[1], out) && threadIdx.x == 0) {
    if (st->nranks > 1) {
      st->local[1] = out[0];
      st->local[2] = out[1];
    } else {
      finish_beta(st, out[0], out[1]);
    }
  }
}

// p = dinv r + beta p
__global__ void __launch_bounds__(kThreads) k_direction(double* __restrict__ p, const double* __restrict__ r,
                                                        const double* __restrict__ dinv, int64_t n, PcgState* st) {
  if (ld_cg(&st->done_d) != 0.0) return;
  const double beta = ld_cg(&st->beta);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    p[k] = fma(beta, p[k], dinv[k] * r[k]);
}

// r = f - q (q = K x0, or q == nullptr for x0 = 0); z = dinv r; p = z; partial r.z, r.r, f.f.
__global__ void __launch_bounds__(kThreads) k_init(const double* __restrict__ f, const double* __restrict__ q,
                                                   const double* __restrict__ dinv, double* __restrict__ r,
                                                   double* __restrict__ p, int64_t n, PcgState* st, double* part) {
  double rz = 0.0, rr = 0.0, ff = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const double fk = f[k];
    const double rk = q ? fk - q[k] : fk;
    const double zk = dinv[k] * rk;
    r[k] = rk;
    p[k] = zk;
    rz = fma(rk, zk, rz);
    rr = fma(rk, rk, rr);
    ff = fma(fk, fk, ff);
  }
  const double mine[3] = {rz, rr, ff};
  double out[3];
  if (grid_reduce<3>(mine, part, &st->ticket[2], out) && threadIdx.x == 0) {
    if (st->nranks > 1) {
      st->local[0] = out[0];
      st->local[1] = out[1];
      st->local[2] = out[2];
    } else {
      finish_init(st, out[0], out[1], out[2]);
    }
  }
}

// ||f - q||^2 over own rows -> st->local[3] (true residual check).
__global__ void __launch_bounds__(kThreads) k_resid(const double* __restrict__ f, const double* __restrict__ q, int64_t n,
                                                    PcgState* st, double* part) {
  double s = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const double d = f[k] - q[k];
    s = fma(d, d, s);
  }
  const double mine[1] = {s};
  double out[1];
  if (grid_reduce<1>(mine, part, &st->ticket[3], out) && threadIdx.x == 0) st->local[3] = out[0];
}

// Multi-rank: combine per-rank partials gathered in `all[nranks*4]` in rank order.
__global__ void k_combine(PcgState* st, const double* __restrict__ all, int stage) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s[4] = {0, 0, 0, 0};
  for (int r = 0; r < st->nranks; ++r)
    for (int v = 0; v < 4; ++v) s[v] += all[4 * r + v];
  if (stage == 0) finish_init(st, s[0], s[1], s[2]);
  if (stage == 1) {
    if (ld_cg(&st->done_d) != 0.0) return;
    finish_alpha(st, s[0]);
  }
  if (stage == 2) {
    if (ld_cg(&st->done_d) != 0.0) return;
    finish_beta(st, s[1], s[2]);
  }
  if (stage == 3) st->local[3] = s[3];
}

}  // namespace

int pcg_grid() { return 4 * num_sms(); }

void launch_spmv(const int64_t* node_ptr, const int32_t* nbr, const double* vals, int64_t nloc, const double* x_full,
                 int64_t own_off, double* y, PcgState* st, double* part, bool pcg, cudaStream_t s) {
  if (pcg)
    k_spmv<true><<<pcg_grid(), kThreads, 0, s>>>(node_ptr, nbr, vals, nloc, x_full, own_off, y, st, part);
  else
    k_spmv<false><<<pcg_grid(), kThreads, 0, s>>>(node_ptr, nbr, vals, nloc, x_full, own_off, y, st, part);
  FS_LAUNCH_CHECK();
}

void launch_update(double* x, double* r, const double* p, const double* q, const double* dinv, int64_t n, PcgState* st,
                   double* part, cudaStream_t s) {
  k_update<<<pcg_grid(), kThreads, 0, s>>>(x, r, p, q, dinv, n, st, part);
  FS_LAUNCH_CHECK();
}

void launch_direction(double* p, const double* r, const double* dinv, int64_t n, PcgState* st, cudaStream_t s) {
  k_direction<<<pcg_grid(), kThreads, 0, s>>>(p, r, dinv, n, st);
  FS_LAUNCH_CHECK();
}

void launch_init(const double* f, const double* q, const double* dinv, double* r, double* p, int64_t n, PcgState* st,
                 double* part, cudaStream_t s) {
  k_init<<<pcg_grid(), kThreads, 0, s>>>(f, q, dinv, r, p, n, st, part);
  FS_LAUNCH_CHECK();
}

void launch_resid(const double* f, const double* q, int64_t n, PcgState* st, double* part, cudaStream_t s) {
  k_resid<<<pcg_grid(), kThreads, 0, s>>>(f, q, n, st, part);
  FS_LAUNCH_CHECK();
}

void launch_combine(PcgState* st, const double* all, int stage, cudaStream_t s) {
  k_combine<<<1, 32, 0, s>>>(st, all, stage);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
