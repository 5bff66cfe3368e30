// Small-mesh PCG in ONE launch of one thread-block cluster (SURVEY.md §3 device-side loop,
// S8-S9; cfg1-3 were launch-bound at 12-16 us per iteration).
//
// CTA c of the cluster owns the node rows [split[c], split[c+1]) (balanced by stored + transposed
// blocks).  Per iteration, with the standard Jacobi-PCG recurrence (PAPER.md:365 / reading Q9):
//   q = K p on the own rows (half-warp per node, gather form of the symmetric storage), p.q partial;
//   cluster barrier; every CTA sums the C partials over distributed shared memory in rank order
//     -> alpha = rho / p.q (identical in every CTA: the decisions below are uniform);
//   x += alpha p, r -= alpha q, z = D^-1 r on the own dofs (z kept in q), r.r and r.z partials;
//   cluster barrier; sums in rank order -> stop tests, beta = rz / rho;
//   p = z + beta p on the own dofs; cluster barrier (release / acquire: the next product reads
//   every CTA's p from L2, with L1-bypassing loads).
// No host round trip and no kernel boundary inside the solve; every sum has a fixed order, so the
// result is bitwise reproducible (it differs in rounding from the multi-kernel path, whose
// reductions are grouped differently).
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "pcg.cuh"

namespace fsfem {
namespace cg = cooperative_groups;

namespace {

#ifndef FSFEM_CL_THREADS
#define FSFEM_CL_THREADS 512
#endif
#ifndef FSFEM_CL_ITEMS
#define FSFEM_CL_ITEMS 6
#endif
constexpr int kCThreads = FSFEM_CL_THREADS;
constexpr int kCWarps = kCThreads / 32;
constexpr int kIt = FSFEM_CL_ITEMS;  // SpMV items per lane per round (16 lanes per node)

// Block sum in a fixed order, returned to every thread.
__device__ __forceinline__ double cta_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // sh may still be read by the previous call
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll 4
  for (int k = 0; k < kCWarps; ++k) t += sh[k];
  return t;
}

// Two block sums with one pair of barriers.
__device__ __forceinline__ void cta_sum2(double& a, double& b, double* sh /*[2 * kCWarps]*/) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    sh[threadIdx.x >> 5] = a;
    sh[kCWarps + (threadIdx.x >> 5)] = b;
  }
  __syncthreads();
  double ta = 0.0, tb = 0.0;
#pragma unroll 4
  for (int k = 0; k < kCWarps; ++k) {
    ta += sh[k];
    tb += sh[kCWarps + k];
  }
  a = ta;
  b = tb;
}

// Sum over the cluster's CTAs, in rank order, of slot `k` of every CTA's red[]: lane c of each
// warp loads CTA c's value over DSMEM, then the warp adds them in sequence.
__device__ __forceinline__ double cluster_sum(cg::cluster_group& cl, double* red, int k, unsigned nr) {
  const unsigned lane = threadIdx.x & 31;
  double v = 0.0;
  for (unsigned base = 0; base < nr; base += 32) {
    const unsigned c = base + lane;
    const double mine = c < nr ? *cl.map_shared_rank(red + k, c) : 0.0;
    const unsigned m = min(32u, nr - base);
    for (unsigned j = 0; j < m; ++j) v += __shfl_sync(0xffffffffu, mine, j);
  }
  return v;
}

__global__ void __launch_bounds__(kCThreads, 1) k_pcg_cluster(
    const int64_t* __restrict__ sptr, const int32_t* __restrict__ snbr, const int64_t* __restrict__ tptr,
    const int2* __restrict__ tlist, const double* __restrict__ vals, const double* __restrict__ dinv,
    double* __restrict__ x, double* __restrict__ r, double* p, double* __restrict__ q,
    const int64_t* __restrict__ split, PcgState* st) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double sh[2 * kCWarps];
  __shared__ double red[4];  // this CTA's partials: p.q, r.r, r.z
  const unsigned rank = cl.block_rank(), nr = cl.num_blocks();
  const int64_t i0 = split[rank], i1 = split[rank + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (__ldcg(&st->done_d) != 0.0) return;  // uniform (written before the launch)
  double rho = __ldcg(&st->rho);
  const double ff = __ldcg(&st->ff), tol = __ldcg(&st->tol);
  long long iters = st->iters;
  const long long max_iter = st->max_iter;
  double alpha = 0.0, beta = 0.0, rr = __ldcg(&st->rr), pq = 0.0;
  int status = FSFEM_OK;
  for (;;) {
    // ---- q = K p on the own rows, p.q ----
    // Half-warp per node, up to kIt (block, component) items per lane per round: every column /
    // list index of the round is loaded first, then every value and p entry, then the FMAs, so a
    // round costs two dependent L2 latencies.
    double dot = 0.0;
    for (int64_t base = i0 + 2 * w; base < i1; base += 2 * kCWarps) {
      const int64_t il = base + (lane >> 4);
      const bool act = il < i1;
      const int gl = lane & 15;
      const int64_t Ps = act ? sptr[il] : 0, Pt = act ? tptr[il] : 0;
      const int nus = act ? static_cast<int>(3 * (sptr[il + 1] - Ps)) : 0;
      const int ntot = act ? nus + static_cast<int>(3 * (tptr[il + 1] - Pt)) : 0;
      int rounds = (ntot + 16 * kIt - 1) / (16 * kIt);
      rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, 16));
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int rd = 0; rd < rounds; ++rd) {
        int64_t vb[kIt];  // index of the first value, stride (3: stored column, 1: transposed row)
        int64_t xi[kIt];
        int vs[kIt];
#pragma unroll
        for (int u = 0; u < kIt; ++u) {
          const int k = 16 * (kIt * rd + u) + gl;
          vb[u] = -1;
          xi[u] = 0;
          vs[u] = 3;
          if (k < nus) {
            const int b = k / 3, cc = k - 3 * b;
            vb[u] = 9 * (Ps + b) + cc;
            xi[u] = 3 * static_cast<int64_t>(__ldg(snbr + Ps + b)) + cc;
          } else if (k < ntot) {
            const int kt = k - nus;
            const int b = kt / 3, cc = kt - 3 * b;
            const int2 e = __ldg(tlist + Pt + b);
            vb[u] = 9 * static_cast<int64_t>(e.x) + 3 * cc;
            xi[u] = 3 * static_cast<int64_t>(e.y) + cc;
            vs[u] = 1;
          }
        }
        double v0[kIt], v1[kIt], v2[kIt], xv[kIt];
#pragma unroll
        for (int u = 0; u < kIt; ++u) {
          const bool ok = vb[u] >= 0;
          const double* pb = vals + (ok ? vb[u] : 0);
          v0[u] = ok ? __ldg(pb) : 0.0;
          v1[u] = ok ? __ldg(pb + vs[u]) : 0.0;
          v2[u] = ok ? __ldg(pb + 2 * vs[u]) : 0.0;
          xv[u] = ok ? __ldcg(p + xi[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kIt; ++u) {
          s0 = fma(v0[u], xv[u], s0);
          s1 = fma(v1[u], xv[u], s1);
          s2 = fma(v2[u], xv[u], s2);
        }
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (act && gl == 0) {
        q[3 * il] = s0;
        q[3 * il + 1] = s1;
        q[3 * il + 2] = s2;
        dot = fma(__ldcg(p + 3 * il), s0, dot);
        dot = fma(__ldcg(p + 3 * il + 1), s1, dot);
        dot = fma(__ldcg(p + 3 * il + 2), s2, dot);
      }
    }
    const double pqc = cta_sum(dot, sh);
    if (threadIdx.x == 0) red[0] = pqc;
    cl.sync();
    pq = cluster_sum(cl, red, 0, nr);
    if (!(pq > 0.0) || !isfinite(pq)) {
      status = FSFEM_ERR_BREAKDOWN;
      break;
    }
    alpha = rho / pq;
    // ---- x += alpha p, r -= alpha q, z = D^-1 r (into q), r.r, r.z ----
    double rrp = 0.0, rzp = 0.0;
    for (int64_t k = 3 * i0 + threadIdx.x; k < 3 * i1; k += kCThreads) {
      const double pk = p[k];
      x[k] = fma(alpha, pk, x[k]);
      const double rk = fma(-alpha, q[k], r[k]);
      r[k] = rk;
      const double zk = dinv[k] * rk;
      q[k] = zk;
      rrp = fma(rk, rk, rrp);
      rzp = fma(rk, zk, rzp);
    }
    cta_sum2(rrp, rzp, sh);
    if (threadIdx.x == 0) {
      red[1] = rrp;
      red[2] = rzp;
    }
    cl.sync();
    const double RR = cluster_sum(cl, red, 1, nr), RZ = cluster_sum(cl, red, 2, nr);
    iters += 1;
    rr = RR;
    if (!isfinite(RR) || !isfinite(RZ)) {
      status = FSFEM_ERR_BREAKDOWN;
      break;
    }
    if (sqrt(RR) <= tol * sqrt(ff)) {
      status = FSFEM_OK;
      break;
    }
    if (iters >= max_iter) {
      status = FSFEM_ERR_NOT_CONVERGED;
      break;
    }
    beta = RZ / rho;
    rho = RZ;
    // ---- p = z + beta p ----
    for (int64_t k = 3 * i0 + threadIdx.x; k < 3 * i1; k += kCThreads) p[k] = fma(beta, p[k], q[k]);
    cl.sync();
  }
  cl.sync();  // no CTA leaves while another may still read its shared memory
  if (rank == 0 && threadIdx.x == 0) {
    st->iters = iters;
    st->rr = rr;
    st->rho = rho;
    st->pq = pq;
    st->alpha = alpha;
    st->beta = beta;
    st->status = status;
    st->done_d = 1.0;
  }
}

// split[c] = first own node whose block prefix (stored + transposed) reaches c / C of the total.
__global__ void k_cluster_split(const int64_t* __restrict__ sptr, const int64_t* __restrict__ tptr, int64_t nloc,
                                int C, int64_t* __restrict__ split) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > C) return;
  if (c == 0 || c == C) {
    split[c] = c == 0 ? 0 : nloc;
    return;
  }
  const int64_t total = (sptr[nloc] - sptr[0]) + (tptr[nloc] - tptr[0]);
  const int64_t want = total * c / C;
  int64_t lo = 0, hi = nloc;  // first i with prefix(i) >= want
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((sptr[mid] - sptr[0]) + (tptr[mid] - tptr[0]) >= want) hi = mid;
    else lo = mid + 1;
  }
  split[c] = lo;
}

int g_cluster_max = 0;  // largest launchable cluster of k_pcg_cluster (0: not probed yet)

int cluster_max() {
  if (g_cluster_max == 0) {
    g_cluster_max = 8;  // portable size
    if (cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(kCThreads);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_pcg_cluster, &cfg) == cudaSuccess && n > 0) g_cluster_max = 16;
    }
    cudaGetLastError();
  }
  return g_cluster_max;
}

}  // namespace

int cluster_pcg_size(int64_t nloc) {
  const int64_t want = std::max<int64_t>(1, (nloc + 63) / 64);  // at least one node per half-warp
  return static_cast<int>(std::min<int64_t>(want, cluster_max()));
}

void cluster_pcg_split(const Pattern& pat, int C, int64_t* split, cudaStream_t s) {
  k_cluster_split<<<1, 64, 0, s>>>(pat.sptr.get(), pat.tptr.get(), pat.nloc, C, split);
  FS_LAUNCH_CHECK();
}

void launch_pcg_cluster(const Pattern& pat, const double* vals, const double* dinv, double* x, double* r, double* p,
                        double* q, const int64_t* split, int C, PcgState* st, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FS_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_cluster, pat.sptr.get(), pat.snbr.get(), pat.tptr.get(), pat.tlist.get(),
                             vals, dinv, x, r, p, q, split, st));
  count_launch();
}

}  // namespace fsfem
