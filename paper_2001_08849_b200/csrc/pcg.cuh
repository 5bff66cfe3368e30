// Device-resident PCG scalars and the scalar steps of the recurrence.
#pragma once
#include "common.cuh"
#include <vector>
#include "pattern.cuh"

namespace fsfem {

struct PcgState {
  double rho;       // r.z
  double alpha, beta;
  double rr;        // r.r (recurrence residual squared)
  double ff;        // f.f
  double tol;       // relative tolerance on ||r|| / ||f||
  double pq;        // p.q
  double done_d;    // != 0: stop (converged, breakdown or max_iter)
  double local[4];  // this rank's partial sums (multi-rank) / true residual^2 (slot 3)
  long long iters;
  long long max_iter;
  int status;       // FSFEM_OK, FSFEM_ERR_NOT_CONVERGED or FSFEM_ERR_BREAKDOWN
  int nranks;
  unsigned int ticket[4];
  unsigned int bar_count, bar_gen;  // grid barrier of the fused update/direction kernel
  // single-reduction variant (Chronopoulos-Gear): rho = gamma = r.u,
  // alpha_prev, the partial sums of gamma and r.r written by the update kernel (upd_n CTAs)
  int variant;      // 0: standard recurrence, 1: single reduction per iteration
  int cg_first;     // 1 until the SpMV after the initial residual has set the first alpha
  double alpha_prev;
  const double* upd_part;  // [2 * upd_n]: gamma partials, then r.r partials
  int upd_n;
  int pad_;
  // device timing of the PCG SpMV launches (%globaltimer, ns): spmv_t0 unused, summed durations
  // (CTA 0 start -> last CTA end) and their number
  unsigned long long spmv_t0;
  unsigned long long spmv_ns;
  unsigned long long spmv_cnt;
  double pq_part;  // split SpMV (halo exchange overlap): p.q of the interior chunks
  // FSFEM_GAP_TIMING (tuning builds): end of the last SpMV, update kernel start / duration, gaps
  unsigned long long spmv_tend, upd_t0, upd_ns, gap_ns, upd_cnt;
  unsigned int upd_done;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// SpMV launch timing, fire-and-forget (nothing serial at the end of the launch): CTA 0 adds
// -t_start and the launch's last CTA adds t_end to spmv_ns (mod 2^64, so the sum is exactly the
// summed durations CTA 0 start -> last CTA end), and counts the launch.
#ifndef FSFEM_SPMV_DEVTIME
#define FSFEM_SPMV_DEVTIME 1
#endif
__device__ __forceinline__ void spmv_time_start(PcgState* st) {
  if (FSFEM_SPMV_DEVTIME && st && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long neg = 0ull - global_ns();
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(&st->spmv_ns), "l"(neg) : "memory");
  }
}
__device__ __forceinline__ void spmv_time_end(PcgState* st) {  // one thread of the last CTA
  if (!FSFEM_SPMV_DEVTIME) return;
  const unsigned long long t1 = global_ns();
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(&st->spmv_ns), "l"(t1) : "memory");
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(&st->spmv_cnt), "l"(1ull) : "memory");
  st->spmv_tend = t1;
}

__device__ __forceinline__ void pcg_stop(PcgState* st, int status) {
  st->status = status;
  st->done_d = 1.0;
}

__device__ __forceinline__ void finish_init(PcgState* st, double rz, double rr, double ff) {
  st->rho = rz;
  st->rr = rr;
  st->ff = ff;
  st->iters = 0;
  st->status = FSFEM_OK;
  st->done_d = 0.0;
  if (!isfinite(rz) || !isfinite(rr) || !isfinite(ff)) {
    pcg_stop(st, FSFEM_ERR_BREAKDOWN);
  } else if (ff == 0.0 || sqrt(rr) <= st->tol * sqrt(ff)) {
    pcg_stop(st, FSFEM_OK);
  } else if (st->max_iter <= 0) {
    pcg_stop(st, FSFEM_ERR_NOT_CONVERGED);
  }
}

__device__ __forceinline__ void finish_alpha(PcgState* st, double pq) {
  st->pq = pq;
  if (!(pq > 0.0) || !isfinite(pq)) {
    pcg_stop(st, FSFEM_ERR_BREAKDOWN);
  } else {
    st->alpha = st->rho / pq;
  }
}

__device__ __forceinline__ void finish_beta(PcgState* st, double rr, double rz) {
  st->iters += 1;
  st->rr = rr;
  if (!isfinite(rr) || !isfinite(rz)) {
    pcg_stop(st, FSFEM_ERR_BREAKDOWN);
  } else if (sqrt(rr) <= st->tol * sqrt(st->ff)) {
    pcg_stop(st, FSFEM_OK);
  } else if (st->iters >= st->max_iter) {
    pcg_stop(st, FSFEM_ERR_NOT_CONVERGED);
  } else {
    st->beta = rz / st->rho;
    st->rho = rz;
  }
}

// Single-reduction recurrence, once delta = u.w (w = K u) and the update kernel's sums
// gamma' = r.u and r.r of the same iteration are known (one combined reduction per iteration):
//   first call:  alpha = gamma / delta, beta = 0
//   then:        iters += 1; stop tests on r.r; beta = gamma'/gamma,
//                alpha = gamma' / (delta - beta gamma' / alpha_prev); gamma = gamma'
// (mathematically the PCG recurrence of finish_alpha / finish_beta, with p = u + beta p and
// s = K p carried as w + beta s).
__device__ __forceinline__ void finish_cg(PcgState* st, double delta, double gamma_new, double rr) {
  if (st->cg_first) {
    st->cg_first = 0;
    st->pq = delta;
    if (!(delta > 0.0) || !isfinite(delta)) {
      pcg_stop(st, FSFEM_ERR_BREAKDOWN);
      return;
    }
    st->alpha = st->rho / delta;
    st->beta = 0.0;
    st->alpha_prev = st->alpha;
    return;
  }
  st->iters += 1;
  st->rr = rr;
  if (!isfinite(rr) || !isfinite(gamma_new) || !isfinite(delta)) {
    pcg_stop(st, FSFEM_ERR_BREAKDOWN);
  } else if (sqrt(rr) <= st->tol * sqrt(st->ff)) {
    pcg_stop(st, FSFEM_OK);
  } else if (st->iters >= st->max_iter) {
    pcg_stop(st, FSFEM_ERR_NOT_CONVERGED);
  } else {
    const double beta = gamma_new / st->rho;
    const double den = delta - beta * gamma_new / st->alpha_prev;
    st->pq = den;
    if (!(den > 0.0) || !isfinite(den)) {
      pcg_stop(st, FSFEM_ERR_BREAKDOWN);
      return;
    }
    st->beta = beta;
    st->alpha = gamma_new / den;
    st->alpha_prev = st->alpha;
    st->rho = gamma_new;
  }
}

// Deterministic dots (det.cu): fixed global chunks of this many nodes; partition ranges are
// aligned to it in deterministic mode.
constexpr int64_t kDetChunkNodes = 256;
int64_t det_nchunks(int64_t nn);
// kind 0 init (r.z, r.r, f.f), 1 p.q, 2 update x, r (r.r, r.z), 3 true residual (|f-q|^2, x.x);
// partials of the own rows' chunks into dpart[3 * chunk + v].
void launch_det_dots(int kind, int64_t n_lo, int64_t nloc, const double* f, const double* q, const double* dinv,
                     double* r, double* p, double* x, PcgState* st, double* dpart, cudaStream_t s);
// Sum of all chunk partials in chunk order, then the scalar step (0 init, 1 alpha, 2 beta, 3 resid).
void launch_det_finish(PcgState* st, const double* dpart, int64_t nchg, int stage, cudaStream_t s);
// Canonical-order SpMV (no fused dot): bitwise independent of the partition.
void launch_spmv_canon(const Pattern& pat, const double* vals, const double* x_full, double* y, const PcgState* st,
                       cudaStream_t s);
// 2 * sum of squares of the stored values (bound of ||K||_F^2 of the rank's rows) -> st->local[2].
void launch_sumsq(const double* vals, int64_t n, PcgState* st, double* part, cudaStream_t s);
// Node ranges of the ranks (det.cu), balanced by node-face incidences, aligned to `align`.
void partition_ranges_device(const int32_t* face_nodes, const int32_t* face_opp, int64_t nf, int64_t nn, int nranks,
                             int64_t align, DevBuf<unsigned char>& scratch, cudaStream_t s,
                             std::vector<int64_t>& ranges);

// Device-side loop: sets the while-node condition to "not done" (pcg.cu).
void launch_loop_cond(cudaGraphConditionalHandle h, const PcgState* st, cudaStream_t s);

int pcg_grid();
int spmv_kind(const Pattern& pat);  // 0 small, 1 gather, 2 dataflow (pcg.cu)
// y (own rows) = K x_full; own_off = 3 * n_lo, the offset of the own rows in x_full (the dataflow
// kernel forms K_ij^T x_i from the own slice, PCG also the p.q partial).
void launch_spmv(const Pattern& pat, const double* vals, const double* x_full, int64_t own_off, double* y,
                 PcgState* st, double* part, bool pcg, cudaStream_t s);
// Split PCG SpMV: part 1 = the chunks whose columns are all own rows (they need
// no exchanged entry), part 2 = the others; p.q = part 1 + part 2 in that order (gather kernel).
void launch_spmv_split(const Pattern& pat, int part_no, const double* vals, const double* x_full, int64_t own_off,
                       double* y, PcgState* st, double* part, cudaStream_t s);
// Interior/boundary chunk order for the split SpMV (once per pattern, row partitions).
void build_overlap_chunks(Pattern& pat, cudaStream_t s);
void launch_update(double* x, double* r, const double* p, const double* q, const double* dinv, int64_t n, PcgState* st,
                   double* part, cudaStream_t s);
void launch_direction(double* p, const double* r, const double* dinv, int64_t n, PcgState* st, cudaStream_t s);
// Single-rank: x += alpha p; r -= alpha q; beta; p = dinv r + beta p in one cooperative kernel.
void launch_update_direction(double* x, double* r, double* p, const double* q, const double* dinv, int64_t n,
                             PcgState* st, double* part, cudaStream_t s);
void launch_init(const double* f, const double* q, const double* dinv, double* r, double* p, int64_t n, PcgState* st,
                 double* part, cudaStream_t s);
// ||f - q||^2 -> st->local[3] and ||x||^2 (own rows) -> st->local[1].
void launch_resid(const double* f, const double* q, const double* x, int64_t n, PcgState* st, double* part,
                  cudaStream_t s);
// Multi-rank: per-rank partials all[4 * nranks] summed in rank order, then the scalar step
// (stage 0 init, 1 alpha, 2 beta, 3 true residual, 4 single-reduction, 5 ||K||_F^2 bound).
void launch_combine(PcgState* st, const double* all, int stage, int nranks, cudaStream_t s);
// Single-reduction variant: p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s,
// u = dinv r; per-CTA partials of r.u and r.r into upd_part (no grid-wide step).
void launch_cg_update(double* x, double* r, double* u, double* p, double* sv, const double* w, const double* dinv,
                      int64_t n, PcgState* st, double* upd_part, cudaStream_t s);
int cg_update_grid(int64_t n);

}  // namespace fsfem
