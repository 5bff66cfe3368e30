// S8-S9 — Jacobi-preconditioned CG on the assembled CSR (the paper solves with PARDISO,
// PAPER.md:365/449; the north star replaces it by PCG, reading Q9):
//   r = f - K x0, z = D^-1 r, p = z, rho = r.z
//   loop: q = K p; alpha = rho / p.q; x += alpha p; r -= alpha q;
//         stop if ||r|| <= tol ||f||; z = D^-1 r; rho' = r.z; beta = rho'/rho; p = z + beta p
// Three kernels per iteration (SpMV+dot, update+dots, direction).  Every dot product is a
// fixed-shape tree (warp shuffles, fixed CTA order, "last CTA reduces") so results are
// bitwise reproducible.  Scalars live on the device; the host only polls `done` between
// CUDA-graph batches of iterations.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "pcg.cuh"

namespace fsfem {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// The PCG vectors (x, r, p, q, D^-1; 40 MB at cfg4) are read and written with an L2 evict_last
// hint so that the SpMV's matrix stream (evict_first) does not push them out of L2 between the
// kernels of an iteration (FSFEM_VEC_EVICT_LAST).
#ifndef FSFEM_VEC_EVICT_LAST
#define FSFEM_VEC_EVICT_LAST 1
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_vec(const double* p, uint64_t pol) {
  if (!FSFEM_VEC_EVICT_LAST) return *p;
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_vec(const double* p, uint64_t pol) {  // read-only in the kernel
  if (!FSFEM_VEC_EVICT_LAST) return __ldg(p);
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_vec(double* p, double v, uint64_t pol) {
  if (!FSFEM_VEC_EVICT_LAST) {
    *p = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// Programmatic dependent launch (PDL, FSFEM_PDL): a kernel launched with the programmatic
// serialization attribute may start before its predecessor finished; it waits here before it
// touches anything the predecessor wrote, and the predecessor lets it launch early.
#ifndef FSFEM_PDL
#define FSFEM_PDL 0
#endif
#ifndef FSFEM_COOP
#define FSFEM_COOP 1
#endif
__device__ __forceinline__ void pdl_wait() {
  if (FSFEM_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  if (FSFEM_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// One thread per CTA reads the device-resident PCG scalars (every thread reading the same
// address through L2 would serialise on one L2 slice); the CTA gets them from shared memory.
__device__ __forceinline__ bool cta_scalars(const PcgState* st, const double* field, double& value) {
  __shared__ double sh_s[2];
  if (threadIdx.x == 0) {
    sh_s[0] = ld_cg(&st->done_d);
    sh_s[1] = field ? ld_cg(field) : 0.0;
  }
  __syncthreads();
  value = sh_s[1];
  const bool done = sh_s[0] != 0.0;
  return done;
}

// Deterministic CTA sum of one double per thread (result valid in thread 0).
__device__ __forceinline__ double block_sum(double v, double* sh /*[blockDim / 32]*/) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) r += sh[k];
  __syncthreads();
  return r;
}

// "Last CTA done" pattern: every CTA publishes NV partial sums; the CTA that arrives last sums
// all partials in a fixed tree and returns true (results in out[0..NV) of thread 0).
template <int NV>
__device__ __forceinline__ bool grid_reduce(const double (&mine)[NV], double* part, unsigned int* ticket, double* out) {
  __shared__ double sh[32];
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
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += ld_cg(part + v * gridDim.x + b);
    out[v] = block_sum(s, sh);
  }
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// Last CTA of a PCG SpMV, all threads: dot = p.q (valid in thread 0).  Standard recurrence:
// alpha.  Single-reduction variant: also sums the update kernel's partials of gamma and r.r in
// CTA order (the one combined reduction of the iteration) and runs finish_cg.  Multi-rank: the
// rank's sums go to st->local for the host-side collective.
__device__ void spmv_finish(PcgState* st, double dot) {
  __shared__ double sh_f[32];
  const int variant = st->variant;  // uniform
  if (variant == 0) {
    if (threadIdx.x == 0) {
      if (st->nranks > 1) st->local[0] = dot;
      else finish_alpha(st, dot);
    }
    return;
  }
  const int first = st->cg_first;
  double g = 0.0, rr = 0.0;
  if (!first) {
    const double* up = st->upd_part;
    const int un = st->upd_n;
    for (int k = threadIdx.x; k < un; k += blockDim.x) {
      g += ld_cg(up + k);
      rr += ld_cg(up + un + k);
    }
  }
  g = block_sum(g, sh_f);
  rr = block_sum(rr, sh_f);
  if (threadIdx.x == 0) {
    if (st->nranks > 1) {
      st->local[0] = dot;
      st->local[1] = g;
      st->local[2] = rr;
    } else {
      finish_cg(st, dot, g, rr);
    }
  }
}

// SpMV over the symmetric block storage (pattern.cuh):
//   y_i = sum_{stored j} K_ij x_j + sum_{n_lo <= j < i} K_ji^T x_j.
//
// Streaming design.  The own nodes are cut (once, with the pattern) into chunks of <= 32 nodes
// whose stored blocks and transposed-list entries fit a shared-memory stage.  A persistent CTA
// walks chunks c = blockIdx.x + k*gridDim.x; one thread streams everything contiguous that a
// chunk needs -- node pointers, stored column ids, the transposed list and the stored 3x3 blocks
// (the bulk of the HBM traffic) -- into a 2-stage shared-memory ring with cp.async.bulk
// (TMA bulk copies) completing on an mbarrier, two chunks ahead of the compute.  The compute
// then only gathers x (L1/L2) and the transposed blocks K_ji (L2: row j < i was streamed a
// moment earlier by the wavefront of CTAs).
//
// Compute: warp per node.  A node's blocks are numbered stored first (0..ds-1), then transposed
// (ds..ds+nt-1); block k gives three lane-items (k, c), each one x value times three values:
//   stored block, column c:     y[a] += K_ij[a][c] x_j[c]   (values at 9b + c + 3a, a = 0..2)
//   transposed block, row c:    y[a] += K_ji[c][a] x_j[c]   (values at 9b + 3c + a, a = 0..2)
// Fixed order: per-lane sums in item order, then a fixed warp tree; no atomics.
struct StageLayout {  // every region starts 16-B aligned (cp.async.bulk destinations)
  // byte offsets inside one stage (16-B aligned), sized for the caps plus alignment slack
  static constexpr int kPtr = 0;                                    // kChunkNodes + 4 int64 (sptr)
  static constexpr int kTptr = kPtr + (kChunkNodes + 4) * 8;        // kChunkNodes + 4 int64 (tptr)
  static constexpr int kSnbr = kTptr + (kChunkNodes + 4) * 8;       // kCapBlocks + 4 int32
  static constexpr int kTl = kSnbr + ((kCapBlocks + 4) * 4 + 15) / 16 * 16;  // kCapBlocks + 2 int2
  static constexpr int kVals = kTl + (kCapBlocks + 2) * 8;          // 9 kCapBlocks + 2 double
  static constexpr int kBytes = kVals + (9 * kCapBlocks + 2) * 8;
};
static_assert(StageLayout::kTptr % 16 == 0 && StageLayout::kSnbr % 16 == 0 && StageLayout::kTl % 16 == 0 &&
                  StageLayout::kVals % 16 == 0 && StageLayout::kBytes % 16 == 0,
              "stage regions must be 16-B aligned");
#ifndef FSFEM_SPMV_STAGES
#define FSFEM_SPMV_STAGES 2
#endif
#ifndef FSFEM_SPMV_MINB
#define FSFEM_SPMV_MINB 2
#endif
constexpr int kStages = FSFEM_SPMV_STAGES;
#ifndef FSFEM_SPMV_ITEMS_S
#define FSFEM_SPMV_ITEMS_S 3
#endif
#ifndef FSFEM_SPMV_ITEMS_T
#define FSFEM_SPMV_ITEMS_T 3
#endif
#ifndef FSFEM_SPMV_GROUP
#define FSFEM_SPMV_GROUP 8
#endif
constexpr int kGroupLanes = FSFEM_SPMV_GROUP;  // group mapping: lanes per node
constexpr int kItemsS = FSFEM_SPMV_ITEMS_S;  // group mapping: stored items per lane per round
constexpr int kItemsT = FSFEM_SPMV_ITEMS_T;  // group mapping: transposed items per lane per round
constexpr int kStreamSmem = 128 + 64 + 32 * kStages + kStages * StageLayout::kBytes;  // + alignment slack

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// L2 eviction-priority policies (per-access cache hints).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Copy elements [e0, e1) of a global array (element size `es`) to smem `dst` with 16-B aligned
// source and size; returns the element offset of e0 inside dst and adds the bytes to `tx`.
// The global arrays are allocated with >= 16 B of slack, so the rounded-up tail is readable.
__device__ __forceinline__ int stage_copy(void* dst, const void* base, int64_t e0, int64_t e1, int es, uint64_t* bar,
                                          uint32_t& tx) {
  if (e1 <= e0) return 0;
  const uintptr_t b = reinterpret_cast<uintptr_t>(base);
  const uintptr_t a0 = (b + e0 * es) & ~uintptr_t(15);
  const uintptr_t a1 = (b + e1 * es + 15) & ~uintptr_t(15);
  const uint32_t bytes = static_cast<uint32_t>(a1 - a0);
  bulk_g2s(dst, reinterpret_cast<const void*>(a0), bytes, bar);
  tx += bytes;
  return static_cast<int>((b + e0 * es - a0) / es);
}

__device__ __forceinline__ int stage_copy_hint(void* dst, const void* base, int64_t e0, int64_t e1, int es,
                                               uint64_t* bar, uint32_t& tx, uint64_t pol) {
  if (e1 <= e0) return 0;
  const uintptr_t b = reinterpret_cast<uintptr_t>(base);
  const uintptr_t a0 = (b + e0 * es) & ~uintptr_t(15);
  const uintptr_t a1 = (b + e1 * es + 15) & ~uintptr_t(15);
  const uint32_t bytes = static_cast<uint32_t>(a1 - a0);
  bulk_g2s_hint(dst, reinterpret_cast<const void*>(a0), bytes, bar, pol);
  tx += bytes;
  return static_cast<int>((b + e0 * es - a0) / es);
}

// element offset of element e0 inside its 16-B aligned bulk copy (what stage_copy returns)
__device__ __forceinline__ int stage_off(const void* base, int64_t e0, int es) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(base) + e0 * es;
  return static_cast<int>((a & uintptr_t(15)) / es);
}

struct StageInfo {  // written by the issuing thread, read after the mbarrier wait
  int n0, nn, Ps0, Pt0;
  int dptr, dsn, dtl, dval;  // element offsets of the first needed element in each smem array
};

__device__ __forceinline__ void issue_chunk(const SpmvChunk& ch, const int64_t* sptr, const int64_t* tptr,
                                            const int32_t* snbr, const int2* tlist, const double* vals,
                                            unsigned char* stage, uint64_t* bar, StageInfo* info) {
  uint32_t tx = 0;
  // the expected byte count must be armed before any copy can complete: compute it first
  const int64_t n0 = ch.n0, n1 = ch.n1, Ps0 = ch.Ps0, Ps1 = ch.Ps1, Pt0 = ch.Pt0, Pt1 = ch.Pt1;
  auto rbytes = [](const void* base, int64_t e0, int64_t e1, int es) -> uint32_t {
    if (e1 <= e0) return 0;
    const uintptr_t b = reinterpret_cast<uintptr_t>(base);
    return static_cast<uint32_t>(((b + e1 * es + 15) & ~uintptr_t(15)) - ((b + e0 * es) & ~uintptr_t(15)));
  };
  const uint32_t total = rbytes(sptr, n0, n1 + 1, 8) + rbytes(tptr, n0, n1 + 1, 8) + rbytes(snbr, Ps0, Ps1, 4) +
                         rbytes(tlist, Pt0, Pt1, 8) + rbytes(vals, 9 * Ps0, 9 * Ps1, 8);
  mbar_arrive_expect_tx(bar, total);
  StageInfo in;
  in.n0 = static_cast<int>(n0);
  in.nn = static_cast<int>(n1 - n0);
  in.Ps0 = static_cast<int>(Ps0);
  in.Pt0 = static_cast<int>(Pt0);
  in.dptr = stage_copy(stage + StageLayout::kPtr, sptr, n0, n1 + 1, 8, bar, tx);
  const int dptr_t = stage_copy(stage + StageLayout::kTptr, tptr, n0, n1 + 1, 8, bar, tx);
  (void)dptr_t;  // same parity as dptr: sptr and tptr are both 16-B aligned allocations
  in.dsn = stage_copy(stage + StageLayout::kSnbr, snbr, Ps0, Ps1, 4, bar, tx);
  in.dtl = stage_copy(stage + StageLayout::kTl, tlist, Pt0, Pt1, 8, bar, tx);
  in.dval = stage_copy(stage + StageLayout::kVals, vals, 9 * Ps0, 9 * Ps1, 8, bar, tx);
  *info = in;
}

// q = K p on own rows (+ partial p.q, reduced by the last CTA into alpha).
template <bool kPcg>
__global__ void __launch_bounds__(kThreads, FSFEM_SPMV_MINB) k_spmv(const SpmvChunk* __restrict__ chunks, int nchunks,
                                                       const int64_t* __restrict__ sptr,
                                                       const int64_t* __restrict__ tptr,
                                                       const int32_t* __restrict__ snbr,
                                                       const int2* __restrict__ tlist, const double* __restrict__ vals,
                                                       const double* __restrict__ x, int64_t own_off,
                                                       double* __restrict__ y, PcgState* st, double* part,
                                                       int split = 0) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // the dynamic window follows the static shared memory of grid_reduce: align it by hand
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                      // [kStages]
  StageInfo* infos = reinterpret_cast<StageInfo*>(smem + 64);              // [kStages] (32 B each)
  unsigned char* stages = smem + 64 + 32 * kStages;                         // ring (16-B aligned stages)
  if (kPcg) {
    double unused;
    if (cta_scalars(st, nullptr, unused)) return;
    if (split != 2) spmv_time_start(st);  // split SpMV: one interval from part 1's start to part 2's end
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // chunk walk: grid-strided (contiguous ranges per CTA were slower)
  const int c_first = blockIdx.x, c_end = nchunks, c_step = gridDim.x;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < kStages; ++k) {
      const int c = c_first + k * c_step;
      if (c < c_end)
        issue_chunk(chunks[c], sptr, tptr, snbr, tlist, vals, stages + k * StageLayout::kBytes, &bars[k], &infos[k]);
    }
  }
  double dot = 0.0;
  int it = 0;
#ifndef FSFEM_SPMV_TIMING
#define FSFEM_SPMV_TIMING 0
#endif
#if FSFEM_SPMV_TIMING
  long long t_wait = 0, t_comp = 0, t_sync = 0;
  const long long t_start = clock64();
#endif
  for (int c = c_first; c < c_end; c += c_step, ++it) {
    const int sg = it % kStages;
    SpmvChunk nxt;
    const int cn = c + kStages * c_step;
    if (threadIdx.x == 0 && cn < c_end) nxt = chunks[cn];  // prefetched before the compute
#if FSFEM_SPMV_TIMING
    const long long t0 = clock64();
#endif
    mbar_wait(&bars[sg], (it / kStages) & 1);
#if FSFEM_SPMV_TIMING
    const long long t1 = clock64();
    t_wait += t1 - t0;
#endif
    const unsigned char* stg = stages + sg * StageLayout::kBytes;
    const StageInfo in = infos[sg];
    const int64_t* sp = reinterpret_cast<const int64_t*>(stg + StageLayout::kPtr) + in.dptr;
    const int64_t* tp = reinterpret_cast<const int64_t*>(stg + StageLayout::kTptr) + in.dptr;
    const int32_t* sn = reinterpret_cast<const int32_t*>(stg + StageLayout::kSnbr) + in.dsn;
    const int2* tl = reinterpret_cast<const int2*>(stg + StageLayout::kTl) + in.dtl;
    const double* sv = reinterpret_cast<const double*>(stg + StageLayout::kVals) + in.dval;
    // 8-lane group per node: a warp works on 4 nodes at once, a lane on up to kItemsS + kItemsT
    // independent items per round (loads issued together), then a 3-level group tree.
    constexpr int G = kGroupLanes, NPW = 32 / kGroupLanes;
    const int grp = lane / G, gl = lane % G;
    for (int mb = warp * NPW; mb < in.nn; mb += kWarps * NPW) {
      const int m = mb + grp;
      const bool act = m < in.nn;
      const int ls = act ? static_cast<int>(sp[m]) - in.Ps0 : 0;
      const int ds = act ? static_cast<int>(sp[m + 1] - sp[m]) : 0;
      const int lt = act ? static_cast<int>(tp[m]) - in.Pt0 : 0;
      const int nit = act ? 3 * (ds + static_cast<int>(tp[m + 1] - tp[m])) : 0;
      const int nus = 3 * ds;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      // One round covers kItemsS stored and kItemsT transposed items per lane.  All global
      // gathers of the round (x for stored items; the 3 values of K_ji and x for transposed
      // items) are issued before anything is consumed, and the stored values are read from
      // shared memory only afterwards, so a round costs one memory latency.
      const int nts = nit - nus;
      int rounds = 0;
      while (G * kItemsS * rounds < nus || G * kItemsT * rounds < nts) ++rounds;
#pragma unroll 1
      for (int o = G; o < 32; o <<= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
      for (int r = 0; r < rounds; ++r) {
        double xs[kItemsS], tv[kItemsT][3], xt[kItemsT];
#pragma unroll
        for (int u = 0; u < kItemsS; ++u) {
          const int k = G * (kItemsS * r + u) + gl;
          xs[u] = 0.0;
          if (k < nus) {
            const int b = k / 3, cc = k - 3 * b;
            xs[u] = __ldg(x + 3 * sn[ls + b] + cc);
          }
        }
#pragma unroll
        for (int u = 0; u < kItemsT; ++u) {
          const int k = G * (kItemsT * r + u) + gl;
          tv[u][0] = tv[u][1] = tv[u][2] = xt[u] = 0.0;
          if (k < nts) {
            const int b = k / 3, cc = k - 3 * b;
            const int2 e = tl[lt + b];
            const double* pb = vals + 9 * static_cast<int64_t>(e.x) + 3 * cc;
            tv[u][0] = __ldg(pb);
            tv[u][1] = __ldg(pb + 1);
            tv[u][2] = __ldg(pb + 2);
            xt[u] = __ldg(x + 3 * e.y + cc);
          }
        }
#pragma unroll
        for (int u = 0; u < kItemsS; ++u) {
          const int k = G * (kItemsS * r + u) + gl;
          if (k < nus) {
            const int b = k / 3, cc = k - 3 * b;
            const double* pb = sv + 9 * (ls + b) + cc;
            s0 = fma(pb[0], xs[u], s0);
            s1 = fma(pb[3], xs[u], s1);
            s2 = fma(pb[6], xs[u], s2);
          }
        }
#pragma unroll
        for (int u = 0; u < kItemsT; ++u) {
          s0 = fma(tv[u][0], xt[u], s0);
          s1 = fma(tv[u][1], xt[u], s1);
          s2 = fma(tv[u][2], xt[u], s2);
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (act && gl == 0) {
        const int64_t il = in.n0 + m;
        y[3 * il] = s0;
        y[3 * il + 1] = s1;
        y[3 * il + 2] = s2;
        if (kPcg) {
          const double* xo = x + own_off + 3 * il;
          dot = fma(xo[0], s0, dot);
          dot = fma(xo[1], s1, dot);
          dot = fma(xo[2], s2, dot);
        }
      }
    }
#if FSFEM_SPMV_TIMING
    const long long t2 = clock64();
    t_comp += t2 - t1;
#endif
    __syncthreads();  // every warp is done with this stage
#if FSFEM_SPMV_TIMING
    t_sync += clock64() - t2;
#endif
    if (threadIdx.x == 0 && cn < c_end) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_chunk(nxt, sptr, tptr, snbr, tlist, vals, stages + sg * StageLayout::kBytes, &bars[sg], &infos[sg]);
    }
  }
#if FSFEM_SPMV_TIMING
  if ((threadIdx.x & 31) == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2))
    printf("spmv timing blk %d warp %d: chunks %d total %lld wait %lld comp %lld sync %lld\n", blockIdx.x,
           threadIdx.x >> 5, it, clock64() - t_start, t_wait, t_comp, t_sync);
#endif
  if (!kPcg) return;
  const double mine[1] = {dot};
  double out[1];
  if (grid_reduce<1>(mine, part, &st->ticket[0], out)) {
    // split SpMV: part 1 keeps its p.q, part 2 adds it first (fixed order) and finishes
    if (split == 1) {
      if (threadIdx.x == 0) st->pq_part = out[0];
    } else {
      __shared__ double sh_pq;
      if (threadIdx.x == 0) sh_pq = (split == 2 ? ld_cg(&st->pq_part) : 0.0) + out[0];
      __syncthreads();
      spmv_finish(st, sh_pq);
      if (threadIdx.x == 0) spmv_time_end(st);
    }
  }
}

// Interior chunks of a row partition: every stored column (incl. halo-stored ones) in [lo, hi).
__global__ void k_chunk_interior(const SpmvChunk* __restrict__ chunks, int nch, const int32_t* __restrict__ snbr,
                                 int64_t lo, int64_t hi, int32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nch; c += (gridDim.x * blockDim.x) >> 5) {
    const SpmvChunk ch = chunks[c];
    bool in = true;
    for (int b = ch.Ps0 + lane; b < ch.Ps1; b += 32) {
      const int32_t j = snbr[b];
      in = in && j >= lo && j < hi;
    }
    in = __all_sync(0xffffffffu, in);
    if (lane == 0) flag[c] = in ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------------------------
// Push form of the symmetric product (k_spmv_df below).  For a stored block b = (i, j), j > i,
// the row-i pass already holds K_ij in shared memory and x_i in registers, so it computes the
// transposed product t = K_ij^T x_i there and stores it to tbuf[tpos[b]], the slot of K_ji in
// row j's (contiguous, ascending) transposed list; row j later only sums its slots.  Traffic vs
// the gather kernel: the 72-B K_ji and 24-B x_j gathers of a transposed block become one 24-B
// store and one contiguous 24-B load (L2-resident in between).
struct PushLayout {  // every region 16-B aligned
  static constexpr int kPtr = 0;                                            // kChunkNodes + 4 int64
  static constexpr int kXo = kPtr + (kChunkNodes + 4) * 8;                  // 3 kChunkNodes + 4 double
  static constexpr int kSnbr = kXo + (3 * kChunkNodes + 4) * 8;             // kCapBlocks + 4 int32
  static constexpr int kTp = kSnbr + ((kCapBlocks + 4) * 4 + 15) / 16 * 16;  // kCapBlocks + 4 int32
  static constexpr int kVals = kTp + ((kCapBlocks + 4) * 4 + 15) / 16 * 16;  // 9 kCapBlocks + 2 double
  static constexpr int kBytes = kVals + (9 * kCapBlocks + 2) * 8;
};
static_assert(PushLayout::kXo % 16 == 0 && PushLayout::kSnbr % 16 == 0 && PushLayout::kTp % 16 == 0 &&
                  PushLayout::kVals % 16 == 0 && PushLayout::kBytes % 16 == 0,
              "push stage regions must be 16-B aligned");
#ifndef FSFEM_PUSH_ITEMS
#define FSFEM_PUSH_ITEMS 5
#endif
constexpr int kPushItems = FSFEM_PUSH_ITEMS;
struct PushInfo {
  int n0, nn, Ps0, dptr, dsn, dtp, dval, dxo;
};

__device__ __forceinline__ void issue_chunk_push(const SpmvChunk& ch, const int64_t* sptr, const int32_t* snbr,
                                                 const int32_t* tpos, const double* vals, const double* xown,
                                                 unsigned char* stage, uint64_t* bar, PushInfo* info) {
  uint32_t tx = 0;
  const int64_t n0 = ch.n0, n1 = ch.n1, Ps0 = ch.Ps0, Ps1 = ch.Ps1;
  auto rbytes = [](const void* base, int64_t e0, int64_t e1, int es) -> uint32_t {
    if (e1 <= e0) return 0;
    const uintptr_t b = reinterpret_cast<uintptr_t>(base);
    return static_cast<uint32_t>(((b + e1 * es + 15) & ~uintptr_t(15)) - ((b + e0 * es) & ~uintptr_t(15)));
  };
  const uint32_t total = rbytes(sptr, n0, n1 + 1, 8) + rbytes(snbr, Ps0, Ps1, 4) + rbytes(tpos, Ps0, Ps1, 4) +
                         rbytes(vals, 9 * Ps0, 9 * Ps1, 8) + rbytes(xown, 3 * n0, 3 * n1, 8);
  // the stage description is stored before the arrival, so the phase completion publishes it
  PushInfo in;
  in.n0 = static_cast<int>(n0);
  in.nn = static_cast<int>(n1 - n0);
  in.Ps0 = static_cast<int>(Ps0);
  in.dptr = stage_off(sptr, n0, 8);
  in.dsn = stage_off(snbr, Ps0, 4);
  in.dtp = stage_off(tpos, Ps0, 4);
  in.dval = stage_off(vals, 9 * Ps0, 8);
  in.dxo = stage_off(xown, 3 * n0, 8);
  *info = in;
  mbar_arrive_expect_tx(bar, total);
  // the matrix streams through L2 once per product: evict it first (keeps x and tbuf resident)
  const uint64_t pol = policy_evict_first();
  stage_copy_hint(stage + PushLayout::kPtr, sptr, n0, n1 + 1, 8, bar, tx, pol);
  stage_copy_hint(stage + PushLayout::kSnbr, snbr, Ps0, Ps1, 4, bar, tx, pol);
  stage_copy_hint(stage + PushLayout::kTp, tpos, Ps0, Ps1, 4, bar, tx, pol);
  stage_copy_hint(stage + PushLayout::kVals, vals, 9 * Ps0, 9 * Ps1, 8, bar, tx, pol);
  stage_copy(stage + PushLayout::kXo, xown, 3 * n0, 3 * n1, 8, bar, tx);
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void st_release_cta_s32(int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// ---------------------------------------------------------------------------------------------
// Dataflow push SpMV (one kernel).  Same product and pushes as k_spmv_push; the row sums of the
// pushed products (phase 2) run in the same launch, each chunk as soon as every chunk holding
// one of its producer rows has finished phase 1:
//   compute warps (8):  P1(c) of the CTA's chunks (TMA ring): y'_i into y, pushes into tbuf;
//   loader warp:        the TMA ring; after P1(c) counts c as done for every chunk d that needs
//                       it (c itself and the chunks of its rows' transposed partners; atomic
//                       acq_rel counters).  The CTA whose count completes d queues d;
//   phase-2 warp:       per queued chunk d: y_i = y'_i + sum of row i's tbuf slots (ascending),
//                       the chunk's p.q partial; then the chunk's tbuf lines are dropped from L2
//                       without write-back (they are rewritten before the next read).
// Every sum has a fixed order and the p.q partials are per chunk, reduced in chunk order by the
// last CTA: bitwise reproducible.  Phase-2 warps wait for other CTAs' chunks, so the launch is
// cooperative (every CTA resident); the waits point to chunks whose phase 1 never waits.
#ifndef FSFEM_DF_BATCH
#define FSFEM_DF_BATCH 4
#endif
constexpr int kDfBatch = FSFEM_DF_BATCH;
constexpr int kDfMinChunksPerCta = 16;
#ifndef FSFEM_DF_P2W
#define FSFEM_DF_P2W 1
#endif
#ifndef FSFEM_DF_GREEDY
#define FSFEM_DF_GREEDY 1
#endif
constexpr int kDfP2W = FSFEM_DF_P2W;  // phase-2 warps (2: chunks alternate between them)
static_assert(kDfP2W == 1 || kDfP2W == 2, "one or two phase-2 warps");
constexpr int kDfThreads = kThreads + 32 * (2 + kDfP2W);  // 8 compute warps, loader, counter, phase 2
struct P2Layout {  // phase-2 buffer: node pointers, P1 sums, own x (p.q), pushed slots of one chunk
  static constexpr int kPtr = 0;                               // kChunkNodes + 4 int64
  static constexpr int kY = kPtr + (kChunkNodes + 4) * 8;      // 3 kChunkNodes + 4 double
  static constexpr int kXo = kY + (3 * kChunkNodes + 4) * 8;   // 3 kChunkNodes + 4 double
  static constexpr int kT = kXo + (3 * kChunkNodes + 4) * 8;   // 3 kCapBlocks + 4 double
  static constexpr int kBytes = kT + (3 * kCapBlocks + 4) * 8;
};
static_assert(P2Layout::kY % 16 == 0 && P2Layout::kXo % 16 == 0 && P2Layout::kT % 16 == 0 &&
                  P2Layout::kBytes % 16 == 0,
              "phase-2 buffer regions must be 16-B aligned");
struct P2Info {
  int n0, nn, Pt0, Pt1, dptr, dy, dt, dxo;
};
#ifndef FSFEM_DF_STAGES
#define FSFEM_DF_STAGES 2
#endif
constexpr int kDfStages = FSFEM_DF_STAGES;  // phase-1 TMA ring depth
static_assert(kDfStages >= 2 && kDfStages <= 7, "mbarrier header holds 2 * stages + 2 barriers");
constexpr int kDfHdr = 128 + 32 * kDfStages + 64;  // barriers, stage infos, phase-2 infos
constexpr int kDfPst = (kDfHdr + 127) / 128 * 128;
constexpr int kDfSmem = 128 + kDfPst + kDfStages * PushLayout::kBytes + 2 * P2Layout::kBytes;

template <bool kPcg>
__global__ void __launch_bounds__(kDfThreads, 2) k_spmv_df(
    const SpmvChunk* __restrict__ chunks, int nchunks, const int64_t* __restrict__ sptr,
    const int64_t* __restrict__ tptr, const int32_t* __restrict__ snbr, const int32_t* __restrict__ tpos,
    const double* __restrict__ vals, const int32_t* __restrict__ dep_ptr, const int2* __restrict__ dep_list,
    uint32_t* cnt, uint32_t* ready, double* dotc, uint32_t* sync, double* tbuf,
    const double* __restrict__ x, int64_t own_off, double* y, PcgState* st) {
  static_assert(kChunkNodes <= kWarps * (32 / kGroupLanes), "one pass of the compute warps per chunk");
  static_assert(kChunkNodes <= 32, "phase 2: one lane per node");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  pdl_trigger();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);                     // [kDfStages] P1 stage loaded
  uint64_t* empty = full + kDfStages;                                      // [kDfStages] P1 stage consumed
  uint64_t* p2full = full + 2 * kDfStages;                                 // [2] phase-2 buffer loaded
  PushInfo* pinfo = reinterpret_cast<PushInfo*>(smem + 128);               // [kDfStages]
  P2Info* qinfo = reinterpret_cast<P2Info*>(smem + 128 + 32 * kDfStages);  // [2]
  unsigned char* pst = smem + kDfPst;                                      // kDfStages P1 stages
  unsigned char* qst = pst + kDfStages * PushLayout::kBytes;               // 2 phase-2 buffers
  __shared__ uint32_t sh_epoch;
  __shared__ int sh_done;
  __shared__ int sh_p1done;  // chunks whose phase 1 the loader has seen complete
  __shared__ double sh_p2dot[2];  // p.q of the CTA's chunks, per phase-2 warp (chunk order)
  if (threadIdx.x == 0) {
    for (int k = 0; k < kDfStages; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kWarps);
    }
    for (int k = 0; k < 2; ++k) mbar_init(&p2full[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // everything below may read what the previous kernel wrote
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = nchunks > static_cast<int>(blockIdx.x) ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // the loader's first chunk descriptors are loaded while thread 0 reads the epoch and the done
  // flag (one round trip instead of three in a row before the first bulk copy)
  SpmvChunk pre[kDfStages + 1];
  if (warp == kWarps && lane == 0)
#pragma unroll
    for (int j = 0; j <= kDfStages; ++j) pre[j] = j < K ? chunks[blockIdx.x + j * gridDim.x] : SpmvChunk{};
  if (threadIdx.x == 0) {
    sh_p1done = 0;
    sh_epoch = __ldcg(sync) + 1u;
    sh_done = kPcg ? (ld_cg(&st->done_d) != 0.0) : 0;
  }
  __syncthreads();
  if (sh_done) return;  // uniform over the grid
  if (kPcg) spmv_time_start(st);
  const uint32_t epoch = sh_epoch;
  const double* xown = x + own_off;
#ifndef FSFEM_DF_TIMING
#define FSFEM_DF_TIMING 0
#endif
  long long tA = 0, tB = 0, tC = 0, tq0 = FSFEM_DF_TIMING ? clock64() : 0;
  const long long t_begin = tq0;
  (void)t_begin;
  int nitems = 0;
#define DF_T(acc) if (FSFEM_DF_TIMING) { const long long tq1 = clock64(); acc += tq1 - tq0; tq0 = tq1; }
  if (warp == kWarps) {
    // ---------------- loader warp: P1 stages (TMA ring) ----------------
    SpmvChunk nx = pre[kDfStages];  // (lane 0's copy is the one used)
#pragma unroll
    for (int j = 0; j < kDfStages; ++j)
      if (lane == 0 && j < K)
        issue_chunk_push(pre[j], sptr, snbr, tpos, vals, xown, pst + j * PushLayout::kBytes, &full[j], &pinfo[j]);
    for (int j = 0; j < K; ++j) {
      const int c = blockIdx.x + j * gridDim.x;
      const int sj = j % kDfStages;
      DF_T(tC)
      mbar_wait(&empty[sj], (j / kDfStages) & 1);  // P1(c) done by every compute warp
      DF_T(tA)
      if (lane == 0 && j + kDfStages < K) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_chunk_push(nx, sptr, snbr, tpos, vals, xown, pst + sj * PushLayout::kBytes, &full[sj], &pinfo[sj]);
      }
      if (j + kDfStages + 1 < K) nx = chunks[c + (kDfStages + 1) * gridDim.x];
      if (lane == 0) st_release_cta_s32(&sh_p1done, j + 1);  // -> counter warp
    }
#if defined(FSFEM_DF_STREAMONLY) || defined(FSFEM_DF_P1ONLY)
  } else if (warp > kWarps) {  // timing experiment: no counting, no phase 2
#endif
  } else if (warp == kWarps + 2) {
    // ---------------- counter warp: dependency counts, in batches ----------------
    // A gpu-scope fence costs microseconds under this load, so the warp takes every chunk whose
    // phase 1 is complete (at least one, up to kDfBatch; FSFEM_DF_GREEDY = 0 waits for a full
    // batch: 2 us slower per launch at cfg4) per round: one release fence for all of their writes
    // (ordered before the loader's observation of the mbarriers), relaxed increments, and one
    // acquire fence before the completed chunks are published as ready.
    constexpr int R = 2;  // rounds of 32 dependants per chunk kept in flight (more: slow path)
    int2 e[kDfBatch][R];
    int qq0[kDfBatch], qq1[kDfBatch];
    auto prefetch = [&](int jb) {  // dependants of chunks jb .. jb + kDfBatch - 1
#pragma unroll
      for (int b = 0; b < kDfBatch; ++b) {
        const int c = blockIdx.x + (jb + b) * gridDim.x;
        qq0[b] = jb + b < K ? dep_ptr[c] : 0;
        qq1[b] = jb + b < K ? dep_ptr[c + 1] : 0;
      }
#pragma unroll
      for (int b = 0; b < kDfBatch; ++b)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int q = qq0[b] + 32 * r + lane;
          e[b][r] = q < qq1[b] ? dep_list[q] : make_int2(-1, 1);
        }
    };
    prefetch(0);
    for (int j = 0; j < K;) {
#if FSFEM_DF_GREEDY
      // every chunk complete so far (at least one, at most kDfBatch): no wait for a full batch
      DF_T(tC)
      int avail;
      while ((avail = ld_acquire_cta_s32(&sh_p1done)) <= j) __nanosleep(32);
      const int jd = min(min(K, j + kDfBatch), avail);
#else
      const int jd = min(K, j + kDfBatch);
      DF_T(tC)
      while (ld_acquire_cta_s32(&sh_p1done) < jd) __nanosleep(32);
#endif
      const int nb = jd - j;
      DF_T(tA)
#ifndef FSFEM_DF_NOFENCE
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
      DF_T(tB)
      uint32_t old[kDfBatch][R];
#pragma unroll
      for (int b = 0; b < kDfBatch; ++b)
#pragma unroll
        for (int r = 0; r < R; ++r)
          old[b][r] = b < nb && e[b][r].x >= 0 ? atomicInc(cnt + e[b][r].x, static_cast<uint32_t>(e[b][r].y) - 1u) : 0u;
      for (int b = 0; b < jd - j; ++b)  // dependants beyond R * 32 (rare)
        for (int q = qq0[b] + 32 * R + lane; q < qq1[b]; q += 32) {
          const int2 ee = dep_list[q];
          if (atomicInc(cnt + ee.x, static_cast<uint32_t>(ee.y) - 1u) == static_cast<uint32_t>(ee.y) - 1u) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(ready + ee.x), "r"(epoch) : "memory");
          }
        }
      bool any_last = false;
      int my_ready[kDfBatch * R];
      int nready = 0;
#pragma unroll
      for (int b = 0; b < kDfBatch; ++b)
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (b < nb && e[b][r].x >= 0 && old[b][r] == static_cast<uint32_t>(e[b][r].y) - 1u) {
            my_ready[nready++] = e[b][r].x;
            any_last = true;
          }
      if (jd < K) prefetch(jd);  // in flight during the fence and the next wait
      if (__any_sync(0xffffffffu, any_last)) {
#ifndef FSFEM_DF_NOFENCE
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
        for (int k = 0; k < nready; ++k)
          asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(ready + my_ready[k]), "r"(epoch) : "memory");
      }
      j = jd;
    }
  } else if (warp == kWarps + 1 || (kDfP2W == 2 && warp == kWarps + 3)) {
    // ---------------- phase-2 warp: the CTA's own chunks in order, lane = node ----------------
    // (two phase-2 warps: warp kWarps + 1 takes the even, warp kWarps + 3 the odd chunks, each
    // with its own buffer j & 1 and no prefetch)
    // chunk d's node pointers, pushed slots and P1 sums are bulk-copied into buffer j & 1 once d
    // is ready; the copy of the next chunk is issued before the current one is summed.
    auto ready_now = [&](int d) { return __shfl_sync(0xffffffffu, lane == 0 ? ld_acquire_u32(ready + d) : 0u, 0) == epoch; };
    auto issue = [&](int jj) {
      const int d = blockIdx.x + jj * gridDim.x;
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;\nfence.proxy.async.shared::cta;" ::: "memory");
        const SpmvChunk ch = chunks[d];
        unsigned char* qb = qst + (jj & 1) * P2Layout::kBytes;
        P2Info qi;
        qi.n0 = ch.n0;
        qi.nn = ch.n1 - ch.n0;
        qi.Pt0 = ch.Pt0;
        qi.Pt1 = ch.Pt1;
        qi.dptr = stage_off(tptr, ch.n0, 8);
        qi.dy = stage_off(y, 3 * (int64_t)ch.n0, 8);
        qi.dt = stage_off(tbuf, 3 * (int64_t)ch.Pt0, 8);
        qi.dxo = stage_off(xown, 3 * (int64_t)ch.n0, 8);
        qinfo[jj & 1] = qi;
        auto rbytes = [](const void* base, int64_t e0, int64_t e1, int es) -> uint32_t {
          if (e1 <= e0) return 0;
          const uintptr_t bb = reinterpret_cast<uintptr_t>(base);
          return static_cast<uint32_t>(((bb + e1 * es + 15) & ~uintptr_t(15)) - ((bb + e0 * es) & ~uintptr_t(15)));
        };
        mbar_arrive_expect_tx(&p2full[jj & 1], rbytes(tptr, ch.n0, ch.n1 + 1, 8) +
                                                   rbytes(y, 3 * (int64_t)ch.n0, 3 * (int64_t)ch.n1, 8) +
                                                   (kPcg ? rbytes(xown, 3 * (int64_t)ch.n0, 3 * (int64_t)ch.n1, 8) : 0u) +
                                                   rbytes(tbuf, 3 * (int64_t)ch.Pt0, 3 * (int64_t)ch.Pt1, 8));
        uint32_t tx = 0;
        stage_copy(qb + P2Layout::kPtr, tptr, ch.n0, ch.n1 + 1, 8, &p2full[jj & 1], tx);
        stage_copy(qb + P2Layout::kY, y, 3 * (int64_t)ch.n0, 3 * (int64_t)ch.n1, 8, &p2full[jj & 1], tx);
        stage_copy(qb + P2Layout::kT, tbuf, 3 * (int64_t)ch.Pt0, 3 * (int64_t)ch.Pt1, 8, &p2full[jj & 1], tx);
        if (kPcg) stage_copy(qb + P2Layout::kXo, xown, 3 * (int64_t)ch.n0, 3 * (int64_t)ch.n1, 8, &p2full[jj & 1], tx);
      }
      __syncwarp();
    };
    int issued = 0;
    double p2dot = 0.0;
    const int pw = warp == kWarps + 1 ? 0 : 1;
    for (int j = kDfP2W == 1 ? 0 : pw; j < K; j += kDfP2W) {
      DF_T(tC)
      if (kDfP2W == 2 || issued == j) {  // this chunk's copy must be in flight: wait for it to be ready
        while (!ready_now(blockIdx.x + j * gridDim.x)) __nanosleep(32);
        issue(j);
        ++issued;
      }
      // readiness of the next chunk: the acquire load is issued now and looked at after this
      // chunk's sums, so its latency overlaps them
      uint32_t nflag = 0u;
      const bool probe = kDfP2W == 1 && issued == j + 1 && j + 1 < K;
      if (probe && lane == 0) nflag = ld_acquire_u32(ready + blockIdx.x + (j + 1) * gridDim.x);
      DF_T(tA)
      ++nitems;
      mbar_wait(&p2full[j & 1], (j >> 1) & 1);
      DF_T(tB)
      const unsigned char* qb = qst + (j & 1) * P2Layout::kBytes;
      const P2Info qi = qinfo[j & 1];
      const int64_t* tp = reinterpret_cast<const int64_t*>(qb + P2Layout::kPtr) + qi.dptr;
      const double* yp = reinterpret_cast<const double*>(qb + P2Layout::kY) + qi.dy;
      const double* tv = reinterpret_cast<const double*>(qb + P2Layout::kT) + qi.dt;
      const double* xq = reinterpret_cast<const double*>(qb + P2Layout::kXo) + qi.dxo;
      const bool act = lane < qi.nn;
      const int mm = act ? lane : 0;
      const int e0 = static_cast<int>(tp[mm] - qi.Pt0), e1 = act ? static_cast<int>(tp[mm + 1] - qi.Pt0) : e0;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int e = e0; e < e1; ++e) {
        s0 += tv[3 * e];
        s1 += tv[3 * e + 1];
        s2 += tv[3 * e + 2];
      }
      s0 += yp[3 * mm];
      s1 += yp[3 * mm + 1];
      s2 += yp[3 * mm + 2];
      double dt = 0.0;
      const int64_t il = static_cast<int64_t>(qi.n0) + mm;
      if (act) {
        const uint64_t vpol = policy_evict_last();
        st_vec(y + 3 * il, s0, vpol);
        st_vec(y + 3 * il + 1, s1, vpol);
        st_vec(y + 3 * il + 2, s2, vpol);
        if (kPcg) dt = fma(xq[3 * mm], s0, fma(xq[3 * mm + 1], s1, xq[3 * mm + 2] * s2));
      }
      if (kPcg) {
        dt = warp_sum(dt);
        p2dot += dt;  // this warp's chunks in order (uniform over the warp)
      }
      // the chunk's pushed products are dead: drop their whole L2 lines without write-back
      const uintptr_t lo = reinterpret_cast<uintptr_t>(tbuf + 3 * (int64_t)qi.Pt0);
      const uintptr_t hi = reinterpret_cast<uintptr_t>(tbuf + 3 * (int64_t)qi.Pt1);
      for (uintptr_t ad = ((lo + 127) & ~uintptr_t(127)) + 128 * lane; ad + 128 <= hi; ad += 128 * 32)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(ad) : "memory");
      __syncwarp();
      if (probe && __shfl_sync(0xffffffffu, nflag, 0) == epoch) {
        issue(j + 1);
        ++issued;
      }
    }
    if (kPcg && lane == 0) sh_p2dot[pw] = p2dot;
  } else {
    // ---------------- compute warps: P1 ----------------
#ifdef FSFEM_DF_STREAMONLY
    for (int j = 0; j < K; ++j) {  // timing experiment: consume the stages only
      const int s = j % kDfStages;
      mbar_wait(&full[s], (j / kDfStages) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (K >= 0) return;
#endif
    constexpr int G = kGroupLanes, NPW = 32 / kGroupLanes;
    const int grp = lane / G, gl = lane % G;
    const int m = warp * NPW + grp;  // this group's node inside every chunk
    const uint64_t vpol = policy_evict_last();
    for (int j = 0; j < K; ++j) {
      const int s = j % kDfStages;
      DF_T(tC)
      mbar_wait(&full[s], (j / kDfStages) & 1);
      DF_T(tA)
      const unsigned char* stg = pst + s * PushLayout::kBytes;
      const PushInfo in = pinfo[s];
      const int64_t* sp = reinterpret_cast<const int64_t*>(stg + PushLayout::kPtr) + in.dptr;
      const int32_t* sn = reinterpret_cast<const int32_t*>(stg + PushLayout::kSnbr) + in.dsn;
      const int32_t* tq = reinterpret_cast<const int32_t*>(stg + PushLayout::kTp) + in.dtp;
      const double* sv = reinterpret_cast<const double*>(stg + PushLayout::kVals) + in.dval;
      const double* sx = reinterpret_cast<const double*>(stg + PushLayout::kXo) + in.dxo;
      const bool act = m < in.nn;
      const int mm = act ? m : 0;
      const int ls = act ? static_cast<int>(sp[m]) - in.Ps0 : 0;
      const int nus = act ? 3 * static_cast<int>(sp[m + 1] - sp[m]) : 0;
      const double xi0 = sx[3 * mm], xi1 = sx[3 * mm + 1], xi2 = sx[3 * mm + 2];
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      int rounds = (nus + G * kPushItems - 1) / (G * kPushItems);
#pragma unroll 1
      for (int o = G; o < 32; o <<= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
#ifdef FSFEM_DF_MINWORK
      rounds = 0;  // timing experiment: no per-block work (wrong product)
#endif
      for (int r = 0; r < rounds; ++r) {
        double xs[kPushItems];
#pragma unroll
        for (int u = 0; u < kPushItems; ++u) {
          const int k = G * (kPushItems * r + u) + gl;
          xs[u] = 0.0;
          if (k < nus) {
            const int b = k / 3, cc = k - 3 * b;
#ifdef FSFEM_DF_NOGATHER
            xs[u] = static_cast<double>(sn[ls + b] & 7) + cc;  // timing experiment only (wrong product)
#else
            xs[u] = ldg_vec(x + 3 * sn[ls + b] + cc, vpol);
#endif
          }
        }
#pragma unroll
        for (int u = 0; u < kPushItems; ++u) {
          const int k = G * (kPushItems * r + u) + gl;
          if (k < nus) {
            const int b = k / 3, cc = k - 3 * b;
            const double* pb = sv + 9 * (ls + b) + cc;
            const double v0 = pb[0], v1 = pb[3], v2 = pb[6];
            s0 = fma(v0, xs[u], s0);
            s1 = fma(v1, xs[u], s1);
            s2 = fma(v2, xs[u], s2);
            const int tp = tq[ls + b];
#ifndef FSFEM_DF_NOPUSH
            if (tp >= 0) tbuf[3 * static_cast<int64_t>(tp) + cc] = fma(v2, xi2, fma(v1, xi1, v0 * xi0));
#else
            if (tp == -7) tbuf[0] = v0 * xi0;  // timing experiment: no pushes (wrong product)
#endif
          }
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (act && gl == 0) {
        const int64_t il = static_cast<int64_t>(in.n0) + m;
        y[3 * il] = s0;
        y[3 * il + 1] = s1;
        y[3 * il + 2] = s2;
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");  // phase 2 reads them with bulk copies
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
#if FSFEM_DF_TIMING
  if (lane == 0 && (warp == 0 || warp >= kWarps) && (blockIdx.x % 37) == 0)
    printf("df blk %d %s K %d items %d: A %lld B %lld C %lld end %lld\n", blockIdx.x,
           warp == kWarps ? "load" : (warp == kWarps + 1 || warp == kWarps + 3 ? "p2" : (warp > kWarps ? "count" : "comp")),
           K, nitems, tA, tB, tC, clock64() - t_begin);
#endif
  // last CTA out: advances the epoch; PCG: p.q = the CTAs' partials (each the sum of its chunks'
  // partials in chunk order) summed in CTA order -- a fixed order for the launch's fixed grid
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    if (kPcg) dotc[blockIdx.x] = kDfP2W == 1 ? sh_p2dot[0] : sh_p2dot[0] + sh_p2dot[1];
    __threadfence();
    last = atomicAdd(sync + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (kPcg) {
    __shared__ double sh[32];
    double a = 0.0;
    for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += blockDim.x) a += __ldcg(dotc + b);
    const double pq = block_sum(a, sh);
    spmv_finish(st, pq);
    if (threadIdx.x == 0) spmv_time_end(st);
  }
  if (threadIdx.x == 0) {
    sync[1] = 0u;
    __threadfence();
    atomicExch(sync, epoch);
  }
}

// Small meshes (fewer chunks than SMs: the configurations whose PCG is launch-latency bound):
// a plain warp-per-node kernel without the TMA pipeline -- no mbarrier set-up, no staging, one
// node per warp with all its loads issued directly.  Same items and fixed warp-tree order as
// the group mapping (the choice depends only on the mesh, so results stay reproducible).
template <bool kPcg>
__global__ void __launch_bounds__(kThreads) k_spmv_small(const int64_t* __restrict__ sptr,
                                                         const int32_t* __restrict__ snbr,
                                                         const int64_t* __restrict__ tptr,
                                                         const int2* __restrict__ tlist,
                                                         const double* __restrict__ vals, int64_t nloc,
                                                         const double* __restrict__ x, int64_t own_off,
                                                         double* __restrict__ y, PcgState* st, double* part) {
  if (kPcg) {
    double unused;
    if (cta_scalars(st, nullptr, unused)) return;
    spmv_time_start(st);
  }
  const int lane = threadIdx.x & 31;
  double dot = 0.0;
  for (int64_t il = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; il < nloc;
       il += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t Ps = sptr[il], Pt = tptr[il];
    const int nus = static_cast<int>(3 * (sptr[il + 1] - Ps));
    const int ntot = nus + static_cast<int>(3 * (tptr[il + 1] - Pt));
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = lane; k < ntot; k += 32) {
      double v0, v1, v2, xv;
      if (k < nus) {
        const int b = k / 3, cc = k - 3 * b;
        const double* pb = vals + 9 * (Ps + b) + cc;
        v0 = __ldg(pb);
        v1 = __ldg(pb + 3);
        v2 = __ldg(pb + 6);
        xv = __ldg(x + 3 * static_cast<int64_t>(__ldg(snbr + Ps + b)) + cc);
      } else {
        const int kt = k - nus;
        const int b = kt / 3, cc = kt - 3 * b;
        const int2 e = __ldg(tlist + Pt + b);
        const double* pb = vals + 9 * static_cast<int64_t>(e.x) + 3 * cc;
        v0 = __ldg(pb);
        v1 = __ldg(pb + 1);
        v2 = __ldg(pb + 2);
        xv = __ldg(x + 3 * static_cast<int64_t>(e.y) + cc);
      }
      s0 = fma(v0, xv, s0);
      s1 = fma(v1, xv, s1);
      s2 = fma(v2, xv, s2);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      y[3 * il] = s0;
      y[3 * il + 1] = s1;
      y[3 * il + 2] = s2;
      if (kPcg) {
        const double* xo = x + own_off + 3 * il;
        dot = fma(xo[0], s0, dot);
        dot = fma(xo[1], s1, dot);
        dot = fma(xo[2], s2, dot);
      }
    }
  }
  if (!kPcg) return;
  const double mine[1] = {dot};
  double out[1];
  if (grid_reduce<1>(mine, part, &st->ticket[0], out)) {
    spmv_finish(st, out[0]);
    if (threadIdx.x == 0) spmv_time_end(st);
  }
}

// Vector kernels: each thread takes kVec elements per pass at stride gridDim*blockDim (coalesced)
// and issues all their loads before any arithmetic, so that enough bytes are in flight to
// stream HBM.  Per-thread partial sums run in element order: the result depends only on the
// (fixed) launch shape.
constexpr int kVec = 4;

// x += alpha p; r -= alpha q; partial r.r and r.z with z = dinv r.
__global__ void __launch_bounds__(kThreads) k_update(double* __restrict__ x, double* __restrict__ r,
                                                     const double* __restrict__ p, const double* __restrict__ q,
                                                     const double* __restrict__ dinv, int64_t n, PcgState* st,
                                                     double* part) {
  double alpha;
  if (cta_scalars(st, &st->alpha, alpha)) return;
  double rr = 0.0, rz = 0.0;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += kVec * T) {
    double xv[kVec], rv[kVec], pv[kVec], qv[kVec], dv[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t k = b + j * T;
      const bool ok = k < n;
      xv[j] = ok ? x[k] : 0.0;
      rv[j] = ok ? r[k] : 0.0;
      pv[j] = ok ? p[k] : 0.0;
      qv[j] = ok ? q[k] : 0.0;
      dv[j] = ok ? dinv[k] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t k = b + j * T;
      if (k < n) {
        x[k] = fma(alpha, pv[j], xv[j]);
        const double rk = fma(-alpha, qv[j], rv[j]);
        r[k] = rk;
        rr = fma(rk, rk, rr);
        rz = fma(rk, dv[j] * rk, rz);
      }
    }
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
  double beta;
  if (cta_scalars(st, &st->beta, beta)) return;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += kVec * T) {
    double pv[kVec], rv[kVec], dv[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t k = b + j * T;
      const bool ok = k < n;
      pv[j] = ok ? p[k] : 0.0;
      rv[j] = ok ? r[k] : 0.0;
      dv[j] = ok ? dinv[k] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t k = b + j * T;
      if (k < n) p[k] = fma(beta, pv[j], dv[j] * rv[j]);
    }
  }
}

// Single-reduction variant (f1): one pass, no grid-wide step (alpha, beta were set by the last
// SpMV).  Per-thread partials in element order, CTA sums into upd_part (reduced by the SpMV's
// last CTA together with u.w).
__global__ void __launch_bounds__(kThreads) k_cg_update(double* __restrict__ x, double* __restrict__ r,
                                                        double* __restrict__ u, double* __restrict__ p,
                                                        double* __restrict__ sv, const double* __restrict__ w,
                                                        const double* __restrict__ dinv, int64_t n, PcgState* st,
                                                        double* __restrict__ upd_part) {
  __shared__ double sh[32];
  __shared__ double sh_sc[3];
  if (threadIdx.x == 0) {
    sh_sc[0] = ld_cg(&st->done_d);
    sh_sc[1] = ld_cg(&st->alpha);
    sh_sc[2] = ld_cg(&st->beta);
  }
  __syncthreads();
  if (sh_sc[0] != 0.0) return;
  const double alpha = sh_sc[1], beta = sh_sc[2];
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  double g = 0.0, rr = 0.0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += kVec * T) {
    double uv[kVec], wv[kVec], pv[kVec], sv_[kVec], xv[kVec], rv[kVec], dv[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t k = b + j * T;
      const bool ok = k < n;
      uv[j] = ok ? u[k] : 0.0;
      wv[j] = ok ? w[k] : 0.0;
      pv[j] = ok ? p[k] : 0.0;
      sv_[j] = ok ? sv[k] : 0.0;
      xv[j] = ok ? x[k] : 0.0;
      rv[j] = ok ? r[k] : 0.0;
      dv[j] = ok ? dinv[k] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t k = b + j * T;
      if (k < n) {
        const double pk = fma(beta, pv[j], uv[j]);
        const double sk = fma(beta, sv_[j], wv[j]);
        const double rk = fma(-alpha, sk, rv[j]);
        const double zk = dv[j] * rk;
        p[k] = pk;
        sv[k] = sk;
        x[k] = fma(alpha, pk, xv[j]);
        r[k] = rk;
        u[k] = zk;
        g = fma(rk, zk, g);
        rr = fma(rk, rk, rr);
      }
    }
  }
  const double tg = block_sum(g, sh), trr = block_sum(rr, sh);
  if (threadIdx.x == 0) {
    upd_part[blockIdx.x] = tg;
    upd_part[gridDim.x + blockIdx.x] = trr;
  }
}

// Single-rank fused update + direction (cooperative launch: all CTAs are co-resident).
//   phase 1: r -= alpha q, per-CTA partials of r.r and r.z (z = dinv r);
//   grid barrier;
//   every CTA sums the partials in the same fixed order (so all agree on beta bit for bit);
//   CTA 0 records the scalars (finish_beta);
//   phase 2: x += alpha p_old; p = dinv r + beta p_old (r and dinv are L2-warm from phase 1).
// Same arithmetic as k_update + k_direction, one launch and one DRAM pass less over r and dinv.
// Grid barrier (every CTA resident): one release atomic per CTA and acquire polls; CTA 0 adds
// 2^31 - (G - 1), the others 1, so bit 31 of the counter flips exactly when all G have arrived and
// its low bits return to 0 (no reset, no generation word, nothing serial after the last arrival).
__device__ __forceinline__ void grid_barrier(PcgState* st) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
    unsigned old, cur;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(&st->bar_count), "r"(inc) : "memory");
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&st->bar_count) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0u);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_update_direction(double* __restrict__ x, double* __restrict__ r,
                                                               double* __restrict__ p, const double* __restrict__ q,
                                                               const double* __restrict__ dinv, int64_t n,
                                                               PcgState* st, double* part) {
  __shared__ double sh[kWarps];
  __shared__ double sh_sc[4];
  pdl_trigger();
  pdl_wait();
#ifndef FSFEM_GAP_TIMING
#define FSFEM_GAP_TIMING 0
#endif
  if (FSFEM_GAP_TIMING && threadIdx.x == 0) atomicMin(&st->upd_t0, global_ns());
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const uint64_t pol = policy_evict_last();
  double rr = 0.0, rz = 0.0;
  // Small enough (<= kKeep passes per thread, cfg4): every load -- r, q, D^-1 and also x, p -- is
  // issued before the grid barrier and z = D^-1 r, x, p stay in registers across it, so phase 2
  // only stores (64 instead of 80 B per dof, no load after the barrier).
#ifndef FSFEM_UPD_KEEP
#define FSFEM_UPD_KEEP 2
#endif
  constexpr int kKeep = FSFEM_UPD_KEEP;
  const bool keep = n <= static_cast<int64_t>(kKeep) * kVec * T;
  double zk_[kKeep][kVec], xk_[kKeep][kVec], pk_[kKeep][kVec];
  // the first pass's loads are issued before the scalars are read, so the two latencies overlap
  // (the loads are only wasted in the launches after convergence)
  double rv0[kVec], qv0[kVec], dv0[kVec];
  if (keep) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t k = b + j * T;
      const bool ok = k < n;
      rv0[j] = ok ? ld_vec(r + k, pol) : 0.0;
      qv0[j] = ok ? ldg_vec(q + k, pol) : 0.0;
      dv0[j] = ok ? ldg_vec(dinv + k, pol) : 0.0;
      xk_[0][j] = ok ? ld_vec(x + k, pol) : 0.0;
      pk_[0][j] = ok ? ld_vec(p + k, pol) : 0.0;
    }
  }
  if (threadIdx.x == 0) {
    sh_sc[0] = ld_cg(&st->done_d);
    sh_sc[1] = ld_cg(&st->alpha);
    sh_sc[2] = ld_cg(&st->rho);
    sh_sc[3] = ld_cg(&st->ff);
  }
  __syncthreads();
  if (sh_sc[0] != 0.0) return;  // uniform over the grid: done_d is only written between launches
  const double alpha = sh_sc[1], rho_old = sh_sc[2];
  if (keep) {
#pragma unroll
    for (int ps = 0; ps < kKeep; ++ps) {
      const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + static_cast<int64_t>(ps) * kVec * T;
      double rv[kVec], qv[kVec], dv[kVec];
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int64_t k = b + j * T;
        const bool ok = k < n;
        if (ps == 0) {
          rv[j] = rv0[j];
          qv[j] = qv0[j];
          dv[j] = dv0[j];
        } else {
          rv[j] = ok ? ld_vec(r + k, pol) : 0.0;
          qv[j] = ok ? ldg_vec(q + k, pol) : 0.0;
          dv[j] = ok ? ldg_vec(dinv + k, pol) : 0.0;
          xk_[ps][j] = ok ? ld_vec(x + k, pol) : 0.0;
          pk_[ps][j] = ok ? ld_vec(p + k, pol) : 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int64_t k = b + j * T;
        zk_[ps][j] = 0.0;
        if (k < n) {  // same element order and arithmetic as the general path below
          const double rk = fma(-alpha, qv[j], rv[j]);
          st_vec(r + k, rk, pol);
          rr = fma(rk, rk, rr);
          rz = fma(rk, dv[j] * rk, rz);
          zk_[ps][j] = dv[j] * rk;
        }
      }
    }
  } else {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += kVec * T) {
      double rv[kVec], qv[kVec], dv[kVec];
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int64_t k = b + j * T;
        const bool ok = k < n;
        rv[j] = ok ? ld_vec(r + k, pol) : 0.0;
        qv[j] = ok ? ldg_vec(q + k, pol) : 0.0;
        dv[j] = ok ? ldg_vec(dinv + k, pol) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int64_t k = b + j * T;
        if (k < n) {
          const double rk = fma(-alpha, qv[j], rv[j]);
          st_vec(r + k, rk, pol);
          rr = fma(rk, rk, rr);
          rz = fma(rk, dv[j] * rk, rz);
        }
      }
    }
  }
  const double trr = block_sum(rr, sh), trz = block_sum(rz, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = trr;
    part[gridDim.x + blockIdx.x] = trz;
  }
  grid_barrier(st);
  // every CTA: the same fixed-order sums of the partials
  double a = 0.0, c = 0.0;
  for (unsigned k = threadIdx.x; k < gridDim.x; k += kThreads) {
    a += ld_cg(part + k);
    c += ld_cg(part + gridDim.x + k);
  }
  const double RR = block_sum(a, sh), RZ = block_sum(c, sh);
  __shared__ double sh_beta;
  if (threadIdx.x == 0) {
    sh_beta = RZ / rho_old;
    if (blockIdx.x == 0) finish_beta(st, RR, RZ);  // same beta; also sets done / iteration count
  }
  __syncthreads();
  const double beta = sh_beta;
  if (keep) {
#pragma unroll
    for (int ps = 0; ps < kKeep; ++ps) {
      const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + static_cast<int64_t>(ps) * kVec * T;
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int64_t k = b + j * T;
        if (k < n) {
          st_vec(x + k, fma(alpha, pk_[ps][j], xk_[ps][j]), pol);
          st_vec(p + k, fma(beta, pk_[ps][j], zk_[ps][j]), pol);
        }
      }
    }
  } else {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += kVec * T) {
      double xv[kVec], pv[kVec], rv[kVec], dv[kVec];
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int64_t k = b + j * T;
        const bool ok = k < n;
        xv[j] = ok ? ld_vec(x + k, pol) : 0.0;
        pv[j] = ok ? ld_vec(p + k, pol) : 0.0;
        rv[j] = ok ? ld_vec(r + k, pol) : 0.0;
        dv[j] = ok ? ldg_vec(dinv + k, pol) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int64_t k = b + j * T;
        if (k < n) {
          st_vec(x + k, fma(alpha, pv[j], xv[j]), pol);
          st_vec(p + k, fma(beta, pv[j], dv[j] * rv[j]), pol);
        }
      }
    }
  }
  if (FSFEM_GAP_TIMING) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&st->upd_done, 1u) == gridDim.x - 1) {
        const unsigned long long t1 = global_ns(), t0 = atomicExch(&st->upd_t0, ~0ull);
        st->upd_ns += t1 - t0;
        if (t0 > st->spmv_tend) st->gap_ns += t0 - st->spmv_tend;
        st->upd_cnt += 1;
        st->upd_done = 0u;
      }
    }
  }
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

// ||f - q||^2 over own rows -> st->local[3] (true residual check), ||x||^2 -> st->local[1].
__global__ void __launch_bounds__(kThreads) k_resid(const double* __restrict__ f, const double* __restrict__ q,
                                                    const double* __restrict__ x, int64_t n, PcgState* st,
                                                    double* part) {
  double s = 0.0, xx = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const double d = f[k] - q[k];
    s = fma(d, d, s);
    xx = fma(x[k], x[k], xx);
  }
  const double mine[2] = {s, xx};
  double out[2];
  if (grid_reduce<2>(mine, part, &st->ticket[3], out) && threadIdx.x == 0) {
    st->local[3] = out[0];
    st->local[1] = out[1];
  }
}

// Multi-rank: combine per-rank partials gathered in `all[nranks*4]` in rank order.
__global__ void k_combine(PcgState* st, const double* __restrict__ all, int stage, int nranks) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s[4] = {0, 0, 0, 0};
  for (int r = 0; r < nranks; ++r)
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
  if (stage == 3) {  // true residual, ||x||^2, ||K||_F^2 bound
    st->local[1] = s[1];
    st->local[2] = s[2];
    st->local[3] = s[3];
  }
  if (stage == 5) st->local[2] = s[2];  // ||K||_F^2 bound only (deterministic mode)
  if (stage == 4) {  // single-reduction variant: (u.w, gamma', r.r) in one collective
    if (ld_cg(&st->done_d) != 0.0) return;
    finish_cg(st, s[0], s[1], s[2]);
  }
}

}  // namespace

int pcg_grid() { return 4 * num_sms(); }
// Small problems: fewer CTAs (less launch, barrier and last-CTA reduction work per iteration).
// The grid only depends on the problem size, so reductions keep a fixed order for a given mesh.
int vec_grid(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(pcg_grid(), ceil_div(n, kThreads * kVec))));
}

int df_grid() {
  static int g = 0;
  if (g == 0) {
    int per_sm = 0;
    FS_CUDA(cudaFuncSetAttribute(k_spmv_df<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDfSmem));
    FS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_df<true>, kDfThreads, kDfSmem));
    g = std::max(1, per_sm) * num_sms();
  }
  return g;
}

int spmv_grid(int64_t nchunks) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(FSFEM_SPMV_MINB * num_sms(), nchunks)));
}

// 0: k_spmv_small (fewer chunks than SMs), 1: k_spmv (gather), 2: k_spmv_df (dataflow push).
// FSFEM_SPMV_KERNEL (tuning / tests) = "gather" or "dataflow" forces 1 or 2 on large meshes; by
// default the dataflow kernel runs when the pattern allows it and every CTA gets enough chunks to
// amortise its pipeline.  The choice depends only on the mesh: results stay reproducible.
int spmv_kind(const Pattern& pat) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = std::getenv("FSFEM_SPMV_KERNEL");
    forced = !e ? 0 : (std::strcmp(e, "gather") == 0 ? 1 : (std::strcmp(e, "dataflow") == 0 ? 2 : 0));
    FS_CUDA(cudaFuncSetAttribute(k_spmv_df<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDfSmem));
    FS_CUDA(cudaFuncSetAttribute(k_spmv_df<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDfSmem));
  }
#ifndef FSFEM_SMALL_CHUNKS_PER_SM
#define FSFEM_SMALL_CHUNKS_PER_SM 1
#endif
  if (pat.nchunks < FSFEM_SMALL_CHUNKS_PER_SM * num_sms()) return 0;
  if (forced == 1 || !pat.df_ok) return 1;
  if (forced == 2) return 2;
  return pat.nchunks >= static_cast<int64_t>(kDfMinChunksPerCta) * df_grid() ? 2 : 1;
}

void launch_spmv(const Pattern& pat, const double* vals, const double* x_full, int64_t own_off, double* y,
                 PcgState* st, double* part, bool pcg, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    FS_CUDA(cudaFuncSetAttribute(k_spmv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem));
    FS_CUDA(cudaFuncSetAttribute(k_spmv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem));
    attr_set = true;
  }
  const int nch = static_cast<int>(pat.nchunks);
  if (spmv_kind(pat) == 0) {  // small mesh: plain warp-per-node kernel
    const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(pcg_grid(), ceil_div(pat.nloc, kWarps))));
    auto kern = pcg ? k_spmv_small<true> : k_spmv_small<false>;
    kern<<<g, kThreads, 0, s>>>(pat.sptr.get(), pat.snbr.get(), pat.tptr.get(), pat.tlist.get(), vals, pat.nloc, x_full,
                                own_off, y, st, part);
    FS_LAUNCH_CHECK();
    return;
  }
  if (spmv_kind(pat) == 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::max(1, std::min(nch, df_grid())));
    cfg.blockDim = dim3(kDfThreads);
    cfg.dynamicSmemBytes = kDfSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;  // phase-2 waits need every CTA resident
    attr[0].val.cooperative = FSFEM_COOP;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = FSFEM_PDL ? 2 : 1;
    const SpmvChunk* chp = pat.chunks.get();
    const int64_t* spp = pat.sptr.get();
    const int64_t* tpp = pat.tptr.get();
    const int32_t* snp = pat.snbr.get();
    const int32_t* tps = pat.tpos.get();
    const int32_t* dpp = pat.dep_ptr.get();
    const int2* dpl = pat.dep_list.get();
    uint32_t* cnt = pat.cnt.get();
    uint32_t* rdy = pat.cflags.get();
    double* dtc = pat.dotc.get();
    uint32_t* syn = pat.sync.get();
    double* tb = pat.tbuf.get();
    if (pcg)
      FS_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_df<true>, chp, nch, spp, tpp, snp, tps, vals, dpp, dpl, cnt, rdy, dtc, syn,
                                 tb, x_full, own_off, y, st));
    else
      FS_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_df<false>, chp, nch, spp, tpp, snp, tps, vals, dpp, dpl, cnt, rdy, dtc, syn,
                                 tb, x_full, own_off, y, st));
    count_launch();
    return;
  }
  if (pcg)
    k_spmv<true><<<spmv_grid(nch), kThreads, kStreamSmem, s>>>(pat.chunks.get(), nch, pat.sptr.get(), pat.tptr.get(),
                                                            pat.snbr.get(), pat.tlist.get(), vals, x_full, own_off, y,
                                                            st, part);
  else
    k_spmv<false><<<spmv_grid(nch), kThreads, kStreamSmem, s>>>(pat.chunks.get(), nch, pat.sptr.get(), pat.tptr.get(),
                                                             pat.snbr.get(), pat.tlist.get(), vals, x_full, own_off, y,
                                                             st, part);
  FS_LAUNCH_CHECK();
}

void build_overlap_chunks(Pattern& pat, cudaStream_t s) {
  FS_CUDA(cudaFuncSetAttribute(k_spmv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem));
  const int64_t nch = pat.nchunks;
  pat.have_ov = true;
  pat.nch_int = 0;
  pat.chunks_ov.ensure(std::max<int64_t>(nch, 1));
  if (nch == 0) return;
  DevBuf<int32_t> flag;
  flag.ensure(nch);
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nch * 32, 256), 16LL * num_sms())));
  k_chunk_interior<<<g, 256, 0, s>>>(pat.chunks.get(), static_cast<int>(nch), pat.snbr.get(), pat.n_lo,
                                     pat.n_lo + pat.nloc, flag.get());
  FS_LAUNCH_CHECK();
  std::vector<int32_t> hf(nch);
  std::vector<SpmvChunk> hc(nch), ho;
  FS_CUDA(cudaMemcpyAsync(hf.data(), flag.get(), sizeof(int32_t) * nch, cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaMemcpyAsync(hc.data(), pat.chunks.get(), sizeof(SpmvChunk) * nch, cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  ho.reserve(nch);
  for (int64_t c = 0; c < nch; ++c)
    if (hf[c]) ho.push_back(hc[c]);
  pat.nch_int = static_cast<int64_t>(ho.size());
  for (int64_t c = 0; c < nch; ++c)
    if (!hf[c]) ho.push_back(hc[c]);
  FS_CUDA(cudaMemcpyAsync(pat.chunks_ov.get(), ho.data(), sizeof(SpmvChunk) * nch, cudaMemcpyHostToDevice, s));
  FS_CUDA(cudaStreamSynchronize(s));
}

void launch_spmv_split(const Pattern& pat, int part_no, const double* vals, const double* x_full, int64_t own_off,
                       double* y, PcgState* st, double* part, cudaStream_t s) {
  const SpmvChunk* ch = pat.chunks_ov.get() + (part_no == 1 ? 0 : pat.nch_int);
  const int n = static_cast<int>(part_no == 1 ? pat.nch_int : pat.nchunks - pat.nch_int);
  // an empty part still runs one CTA: its grid reduction passes the p.q on (part 1) or finishes it
  k_spmv<true><<<std::max(1, spmv_grid(n)), kThreads, kStreamSmem, s>>>(ch, n, pat.sptr.get(), pat.tptr.get(),
                                                                        pat.snbr.get(), pat.tlist.get(), vals, x_full,
                                                                        own_off, y, st, part, part_no);
  FS_LAUNCH_CHECK();
}

void launch_update(double* x, double* r, const double* p, const double* q, const double* dinv, int64_t n, PcgState* st,
                   double* part, cudaStream_t s) {
  k_update<<<vec_grid(n), kThreads, 0, s>>>(x, r, p, q, dinv, n, st, part);
  FS_LAUNCH_CHECK();
}

void launch_direction(double* p, const double* r, const double* dinv, int64_t n, PcgState* st, cudaStream_t s) {
  k_direction<<<vec_grid(n), kThreads, 0, s>>>(p, r, dinv, n, st);
  FS_LAUNCH_CHECK();
}

// Every PCG kernel asks for the same L1/shared-memory split as the SpMV, so that the SMs do not
// reconfigure the carve-out between the kernels of an iteration (FSFEM_CARVEOUT, percent).
#ifndef FSFEM_CARVEOUT
#define FSFEM_CARVEOUT -1
#endif
void set_pcg_carveouts() {
  static bool done = false;
  if (done || FSFEM_CARVEOUT < 0) return;
  done = true;
  const int c = FSFEM_CARVEOUT;
  FS_CUDA(cudaFuncSetAttribute(k_update_direction, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  FS_CUDA(cudaFuncSetAttribute(k_spmv_df<true>, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  FS_CUDA(cudaFuncSetAttribute(k_spmv_df<false>, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  FS_CUDA(cudaFuncSetAttribute(k_update, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  FS_CUDA(cudaFuncSetAttribute(k_direction, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  FS_CUDA(cudaFuncSetAttribute(k_cg_update, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  FS_CUDA(cudaFuncSetAttribute(k_spmv<true>, cudaFuncAttributePreferredSharedMemoryCarveout, c));
  FS_CUDA(cudaFuncSetAttribute(k_spmv_small<true>, cudaFuncAttributePreferredSharedMemoryCarveout, c));
}

int update_direction_grid() {
  static int g = 0;
  set_pcg_carveouts();
  if (g == 0) {
    int per_sm = 0;
    FS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update_direction, kThreads, 0));
#ifndef FSFEM_UPD_PER_SM
#define FSFEM_UPD_PER_SM 4
#endif
    g = std::max(1, std::min(FSFEM_UPD_PER_SM, per_sm)) * num_sms();
  }
  return g;
}

void launch_update_direction(double* x, double* r, double* p, const double* q, const double* dinv, int64_t n,
                             PcgState* st, double* part, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::min(update_direction_grid(), vec_grid(n)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = FSFEM_COOP;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = FSFEM_PDL ? 2 : 1;
  FS_CUDA(cudaLaunchKernelEx(&cfg, k_update_direction, x, r, p, q, dinv, n, st, part));
  count_launch();
}

void launch_init(const double* f, const double* q, const double* dinv, double* r, double* p, int64_t n, PcgState* st,
                 double* part, cudaStream_t s) {
  k_init<<<vec_grid(n), kThreads, 0, s>>>(f, q, dinv, r, p, n, st, part);
  FS_LAUNCH_CHECK();
}

void launch_resid(const double* f, const double* q, const double* x, int64_t n, PcgState* st, double* part,
                  cudaStream_t s) {
  k_resid<<<vec_grid(n), kThreads, 0, s>>>(f, q, x, n, st, part);
  FS_LAUNCH_CHECK();
}

int cg_update_grid(int64_t n) { return vec_grid(n); }

void launch_cg_update(double* x, double* r, double* u, double* p, double* sv, const double* w, const double* dinv,
                      int64_t n, PcgState* st, double* upd_part, cudaStream_t s) {
  k_cg_update<<<cg_update_grid(n), kThreads, 0, s>>>(x, r, u, p, sv, w, dinv, n, st, upd_part);
  FS_LAUNCH_CHECK();
}

// Device-side PCG loop (api.cu): the body of the graph's while node ends with this kernel, which
// keeps the loop running while the recurrence has not stopped.
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const PcgState* st) {
  if (threadIdx.x == 0) cudaGraphSetConditional(h, __ldcg(&st->done_d) == 0.0 ? 1u : 0u);
}

void launch_loop_cond(cudaGraphConditionalHandle h, const PcgState* st, cudaStream_t s) {
  k_loop_cond<<<1, 32, 0, s>>>(h, st);
  FS_LAUNCH_CHECK();
}

void launch_combine(PcgState* st, const double* all, int stage, int nranks, cudaStream_t s) {
  k_combine<<<1, 32, 0, s>>>(st, all, stage, nranks);
  FS_LAUNCH_CHECK();
}

}  // namespace fsfem
