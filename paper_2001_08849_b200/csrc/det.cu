// Row partition helpers and the deterministic (rank-count invariant) PCG reductions
// (SURVEY.md 8(e) "Partition" and "Deterministic option").
//
// Partition: rank r owns the node range [ranges[r], ranges[r+1]).  The ranges balance the
// node-face incidences (sum over the faces of the number of field nodes a rank owns -- the rows'
// share of the assembly work and, through the neighbour count, of the nnz) and are aligned to
// `align` nodes; every rank computes the same ranges from the replicated face table.
//
// Deterministic dots: every dot product of the recurrence is a sum over FIXED global chunks of
// kDetChunkNodes nodes (3 * kDetChunkNodes dofs): each chunk is reduced by one CTA in a fixed
// shape, the chunk partials are exchanged between the ranks (all-gather of each rank's chunk
// range) and every rank sums all of them in global chunk order with the same fixed tree.  With
// ranges aligned to kDetChunkNodes, no chunk straddles two ranks, so the sums -- and with the
// canonical-order SpMV (k_spmv_canon) and the partition-invariant assembly the whole solve --
// are bit-identical for any number of ranks.
#include "common.cuh"
#include "pattern.cuh"
#include "pcg.cuh"

namespace fsfem {

namespace {

constexpr int kT = 256;

__global__ void k_field_count(const int32_t* __restrict__ face_nodes, const int32_t* __restrict__ face_opp, int64_t nf,
                              int32_t* __restrict__ cnt) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) atomicAdd(cnt + face_nodes[3 * f + k], 1);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int32_t v = face_opp[2 * f + k];
      if (v >= 0) atomicAdd(cnt + v, 1);
    }
  }
}

// ranges[r] = the multiple of `align` nearest to the first node whose incidence prefix reaches
// r * total / nranks (monotone, ranges[0] = 0, ranges[nranks] = nn).
__global__ void k_split(const int64_t* __restrict__ pre, int64_t nn, int nranks, int64_t align,
                        int64_t* __restrict__ ranges) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t W = pre[nn];
  ranges[0] = 0;
  for (int r = 1; r < nranks; ++r) {
    const int64_t target = (W * r) / nranks;
    int64_t lo = 0, hi = nn;  // first i with pre[i] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (pre[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    int64_t b = ((lo + align / 2) / align) * align;
    b = b > nn ? nn : b;
    b = b < ranges[r - 1] ? ranges[r - 1] : b;
    ranges[r] = b;
  }
  ranges[nranks] = nn;
}

__device__ __forceinline__ double det_block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < kT / 32; ++k) r += sh[k];
  __syncthreads();
  return r;
}

__device__ __forceinline__ bool det_done(const PcgState* st, double* alpha) {
  __shared__ double sh[2];
  if (threadIdx.x == 0) {
    sh[0] = __ldcg(&st->done_d);
    sh[1] = __ldcg(&st->alpha);
  }
  __syncthreads();
  if (alpha) *alpha = sh[1];
  return sh[0] != 0.0;
}

// One CTA per own global chunk c (dofs [3 kDetChunkNodes c, ...) clipped to [dof_lo, dof_hi));
// thread t takes dofs t, t + 256, t + 512 of the chunk in that order.  Partials -> dpart[3 c + v].
//   kind 0 (init):  r = f - q (q may be null), p = D^-1 r  -> (r.z, r.r, f.f)
//   kind 1 (p.q):                                          -> (p.q, 0, 0)
//   kind 2 (update): x += alpha p, r -= alpha q            -> (r.r, r.z, 0)
//   kind 3 (resid):                                        -> ((f-q).(f-q), x.x, 0)
template <int kKind>
__global__ void __launch_bounds__(kT) k_det_dots(int64_t c0, int64_t dof_lo, int64_t dof_hi, const double* __restrict__ f,
                                                 const double* __restrict__ q, const double* __restrict__ dinv,
                                                 double* __restrict__ r, double* __restrict__ p, double* __restrict__ x,
                                                 PcgState* st, double* __restrict__ dpart) {
  __shared__ double sh[kT / 32];
  double alpha = 0.0;
  if (kKind == 1 || kKind == 2) {
    if (det_done(st, &alpha)) return;
  }
  const int64_t c = c0 + blockIdx.x;
  const int64_t base = 3 * kDetChunkNodes * c;
  double a = 0.0, b = 0.0, e = 0.0;
#pragma unroll
  for (int k = 0; k < 3 * kDetChunkNodes / kT; ++k) {
    const int64_t d = base + threadIdx.x + kT * k;
    if (d < dof_lo || d >= dof_hi) continue;
    const int64_t l = d - dof_lo;  // own-row index
    if (kKind == 0) {
      const double fk = f[l];
      const double rk = q ? fk - q[l] : fk;
      const double zk = dinv[l] * rk;
      r[l] = rk;
      p[l] = zk;
      a = fma(rk, zk, a);
      b = fma(rk, rk, b);
      e = fma(fk, fk, e);
    } else if (kKind == 1) {
      a = fma(p[l], q[l], a);
    } else if (kKind == 2) {
      x[l] = fma(alpha, p[l], x[l]);
      const double rk = fma(-alpha, q[l], r[l]);
      r[l] = rk;
      a = fma(rk, rk, a);
      b = fma(rk, dinv[l] * rk, b);
    } else {
      const double dk = f[l] - q[l];
      a = fma(dk, dk, a);
      b = fma(x[l], x[l], b);
    }
  }
  a = det_block_sum(a, sh);
  b = det_block_sum(b, sh);
  e = det_block_sum(e, sh);
  if (threadIdx.x == 0) {
    dpart[3 * c] = a;
    dpart[3 * c + 1] = b;
    dpart[3 * c + 2] = e;
  }
}

// One CTA: the global sums of the chunk partials in chunk order (fixed tree), then the scalar
// step of the recurrence.  stage 0 init, 1 alpha, 2 beta, 3 true residual (local[3], local[1]).
__global__ void __launch_bounds__(kT) k_det_finish(PcgState* st, const double* __restrict__ dpart, int64_t nchg,
                                                   int stage) {
  __shared__ double sh[kT / 32];
  if ((stage == 1 || stage == 2) && det_done(st, nullptr)) return;
  double s[3] = {0.0, 0.0, 0.0};
  for (int64_t c = threadIdx.x; c < nchg; c += kT)
#pragma unroll
    for (int v = 0; v < 3; ++v) s[v] += __ldcg(dpart + 3 * c + v);
#pragma unroll
  for (int v = 0; v < 3; ++v) s[v] = det_block_sum(s[v], sh);
  if (threadIdx.x != 0) return;
  if (stage == 0) finish_init(st, s[0], s[1], s[2]);
  if (stage == 1) finish_alpha(st, s[0]);
  if (stage == 2) finish_beta(st, s[0], s[1]);
  if (stage == 3) {
    st->local[3] = s[0];
    st->local[1] = s[1];
  }
}

// Canonical-order SpMV (warp per node, no fused dot): row i's 3x3 blocks in ascending column j
// -- stored halo blocks (j < n_lo), then the transposed list (n_lo <= j < i), then the stored
// blocks j >= i -- so the sequence of (block, column) items of a row is the same whatever the
// partition (a halo block K_ij is bitwise K_ji^T).  Item k goes to lane k % 32, per-lane sums in
// item order, fixed warp tree.
__global__ void __launch_bounds__(kT) k_spmv_canon(const int64_t* __restrict__ sptr, const int32_t* __restrict__ snbr,
                                                   const int32_t* __restrict__ sdiag, const int64_t* __restrict__ tptr,
                                                   const int2* __restrict__ tlist, const double* __restrict__ vals,
                                                   int64_t nloc, const double* __restrict__ x, double* __restrict__ y,
                                                   const PcgState* st) {
  if (st) {
    __shared__ double d;
    if (threadIdx.x == 0) d = __ldcg(&st->done_d);
    __syncthreads();
    if (d != 0.0) return;
  }
  const int lane = threadIdx.x & 31;
  for (int64_t il = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; il < nloc;
       il += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t Ps = sptr[il], Pt = tptr[il];
    const int ds = static_cast<int>(sptr[il + 1] - Ps);
    const int nh = sdiag[il];  // stored halo blocks (j < n_lo) precede the diagonal
    const int nt = static_cast<int>(tptr[il + 1] - Pt);
    const int n1 = 3 * nh, n2 = n1 + 3 * nt, ntot = n2 + 3 * (ds - nh);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = lane; k < ntot; k += 32) {
      double v0, v1, v2, xv;
      if (k < n1 || k >= n2) {  // stored block b, column cc: K_ij[a][cc] at 9b + 3a + cc
        const int kk = k < n1 ? k : k - n2 + n1;
        const int b = kk / 3, cc = kk - 3 * b;
        const double* pb = vals + 9 * (Ps + b) + cc;
        v0 = pb[0];
        v1 = pb[3];
        v2 = pb[6];
        xv = x[3 * static_cast<int64_t>(snbr[Ps + b]) + cc];
      } else {  // transposed (K_ji, j), column cc of K_ij = row cc of K_ji
        const int kt = k - n1;
        const int b = kt / 3, cc = kt - 3 * b;
        const int2 e = tlist[Pt + b];
        const double* pb = vals + 9 * static_cast<int64_t>(e.x) + 3 * cc;
        v0 = pb[0];
        v1 = pb[1];
        v2 = pb[2];
        xv = x[3 * static_cast<int64_t>(e.y) + cc];
      }
      s0 = fma(v0, xv, s0);
      s1 = fma(v1, xv, s1);
      s2 = fma(v2, xv, s2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      y[3 * il] = s0;
      y[3 * il + 1] = s1;
      y[3 * il + 2] = s2;
    }
  }
}

// Sum of squares of the stored values (x2: an upper bound of ||K||_F^2 over the rank's rows,
// which only sets the rounding-floor bound of the true residual) -> st->local[2].
__global__ void __launch_bounds__(kT) k_sumsq(const double* __restrict__ vals, int64_t n, PcgState* st,
                                              double* __restrict__ part, unsigned int* ticket) {
  __shared__ double sh[kT / 32];
  __shared__ bool last;
  double s = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    s = fma(vals[k], vals[k], s);
  s = det_block_sum(s, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += kT) t += __ldcg(part + b);
  t = det_block_sum(t, sh);
  if (threadIdx.x == 0) {
    st->local[2] = 2.0 * t;
    *ticket = 0u;
  }
}

}  // namespace

void partition_ranges_device(const int32_t* face_nodes, const int32_t* face_opp, int64_t nf, int64_t nn, int nranks,
                             int64_t align, DevBuf<unsigned char>& scratch, cudaStream_t s,
                             std::vector<int64_t>& ranges) {
  ranges.assign(nranks + 1, 0);
  ranges[nranks] = nn;
  if (nranks == 1) return;
  const size_t tb = scan_tmp_bytes(nn + 1);
  const size_t o_cnt = 0, o_pre = (sizeof(int32_t) * (nn + 1) + 255) & ~size_t(255),
               o_rng = o_pre + ((sizeof(int64_t) * (nn + 1) + 255) & ~size_t(255)),
               o_tmp = o_rng + ((sizeof(int64_t) * (nranks + 1) + 255) & ~size_t(255));
  unsigned char* b = scratch.ensure(o_tmp + tb);
  int32_t* cnt = reinterpret_cast<int32_t*>(b + o_cnt);
  int64_t* pre = reinterpret_cast<int64_t*>(b + o_pre);
  int64_t* rng = reinterpret_cast<int64_t*>(b + o_rng);
  FS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nn + 1), s));
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nf, 256), 8LL * num_sms())));
  k_field_count<<<g, 256, 0, s>>>(face_nodes, face_opp, nf, cnt);
  FS_LAUNCH_CHECK();
  exclusive_scan_i32_to_i64(cnt, pre, nn, s, b + o_tmp, tb);
  k_split<<<1, 32, 0, s>>>(pre, nn, nranks, std::max<int64_t>(1, align), rng);
  FS_LAUNCH_CHECK();
  FS_CUDA(cudaMemcpyAsync(ranges.data(), rng, sizeof(int64_t) * (nranks + 1), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
}

int64_t det_nchunks(int64_t nn) { return ceil_div(nn, kDetChunkNodes); }

// Chunk partials of the own rows [n_lo, n_lo + nloc) (n_lo a multiple of kDetChunkNodes).
void launch_det_dots(int kind, int64_t n_lo, int64_t nloc, const double* f, const double* q, const double* dinv,
                     double* r, double* p, double* x, PcgState* st, double* dpart, cudaStream_t s) {
  if (nloc <= 0) return;
  const int64_t c0 = n_lo / kDetChunkNodes, c1 = ceil_div(n_lo + nloc, kDetChunkNodes);
  const int64_t dlo = 3 * n_lo, dhi = 3 * (n_lo + nloc);
  const int g = static_cast<int>(c1 - c0);
  switch (kind) {
    case 0: k_det_dots<0><<<g, kT, 0, s>>>(c0, dlo, dhi, f, q, dinv, r, p, x, st, dpart); break;
    case 1: k_det_dots<1><<<g, kT, 0, s>>>(c0, dlo, dhi, f, q, dinv, r, p, x, st, dpart); break;
    case 2: k_det_dots<2><<<g, kT, 0, s>>>(c0, dlo, dhi, f, q, dinv, r, p, x, st, dpart); break;
    default: k_det_dots<3><<<g, kT, 0, s>>>(c0, dlo, dhi, f, q, dinv, r, p, x, st, dpart); break;
  }
  FS_LAUNCH_CHECK();
}

void launch_det_finish(PcgState* st, const double* dpart, int64_t nchg, int stage, cudaStream_t s) {
  k_det_finish<<<1, kT, 0, s>>>(st, dpart, nchg, stage);
  FS_LAUNCH_CHECK();
}

void launch_spmv_canon(const Pattern& pat, const double* vals, const double* x_full, double* y, const PcgState* st,
                       cudaStream_t s) {
  if (pat.nloc <= 0) return;
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(32LL * num_sms(), ceil_div(pat.nloc, kT / 32))));
  k_spmv_canon<<<g, kT, 0, s>>>(pat.sptr.get(), pat.snbr.get(), pat.sdiag.get(), pat.tptr.get(), pat.tlist.get(), vals,
                                pat.nloc, x_full, y, st);
  FS_LAUNCH_CHECK();
}

void launch_sumsq(const double* vals, int64_t n, PcgState* st, double* part, cudaStream_t s) {
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4LL * num_sms(), ceil_div(n, kT * 4))));
  k_sumsq<<<g, kT, 0, s>>>(vals, n, st, part, &st->ticket[3]);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
