// C ABI of the FS-FEM hot path (include/fsfem.h): context, call-order state machine,
// host/device pointer handling, stage timing, PCG batching in CUDA graphs, NCCL row partition.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "nccl.h"
#include "pattern.cuh"
#include "pcg.cuh"

namespace fsfem {

// kernels' host drivers (faces.cu, symbolic.cu, assemble.cu, bc.cu)
void build_faces_device(const double* d_xyz, int64_t nn, const int32_t* d_tets, int64_t nt, cudaStream_t s,
                        DevBuf<unsigned char>& scratch, DevBuf<int32_t>& face_nodes, DevBuf<int32_t>& face_tet,
                        DevBuf<int32_t>& face_opp, DevBuf<int32_t>& tet_face, DevBuf<int32_t>& tet_across,
                        int64_t* n_faces, int64_t* n_interior, unsigned long long* h_flags);
void build_pattern_device(const int32_t* d_tets, int64_t nt, const int32_t* tet_face, const int32_t* tet_across,
                          int64_t n_lo, int64_t nloc, cudaStream_t s,
                          DevBuf<unsigned char>& scratch, Pattern& pat, unsigned long long* h_flags, int fem);
void export_csr_device(const Pattern& pat, const double* svals, int64_t* row_ptr, int32_t* col_idx, double* vals,
                       cudaStream_t s);
void face_s_device(const double* xyz, const int32_t* tets, const int32_t* face_nodes, const int32_t* face_tet,
                   const int32_t* face_opp, int64_t nf, double* face_s, double* face_V, cudaStream_t s);
void build_halo_device(Pattern& pat, int64_t nn, const std::vector<int64_t>& ranges, std::vector<int64_t>& need,
                       DevBuf<unsigned char>& scratch, cudaStream_t s);
void halo_pack_device(const double* full, const int32_t* nodes, int64_t n, double* buf, cudaStream_t s);
void halo_unpack_device(const double* buf, const int32_t* nodes, int64_t n, double* full, cudaStream_t s);
void build_assembly_tiles(Pattern& pat, const double* xyz, const int32_t* rec_a, const int32_t* rec_b, bool tet,
                          DevBuf<unsigned char>& scratch, unsigned long long* h_flags, cudaStream_t s);
void assemble_tiles_device(const Pattern& pat, const double* xyz, double lam, double mu, double* vals, bool tet,
                           cudaStream_t s);
void tet_s_device(const double* xyz, const int32_t* tets, int64_t nt, double* tet_s, double* tet_V, cudaStream_t s);
int cluster_pcg_size(int64_t nloc);
void cluster_pcg_split(const Pattern& pat, int C, int64_t* split, cudaStream_t s);
void launch_pcg_cluster(const Pattern& pat, const double* vals, const double* dinv, double* x, double* r, double* p,
                        double* q, const int64_t* split, int C, PcgState* st, cudaStream_t s);
void domain_stiffness_device(const double* xyz, const int32_t* rec_a, const int32_t* rec_b, bool tet,
                             const int64_t* ids, int64_t n, double lam, double mu, double* K, int32_t* field,
                             cudaStream_t s);
void recover_device(const int32_t* rec_a, const int32_t* rec_b, bool tet, const double* rec_s, const double* rec_V,
                    int64_t nrec,
                    const int64_t* nd_ptr, const int32_t* nd_idx, int64_t nloc, const double* u, double lam, double mu,
                    double* strain, double* stress, double* node_stress, double* node_vm, cudaStream_t s);
double mean_tet_span_device(const int32_t* tets, int64_t nt, unsigned long long* d_tmp, cudaStream_t s);
void morton_order_device(const double* d_xyz, int64_t nn, int32_t* iperm, int32_t* perm, DevBuf<unsigned char>& scratch,
                         cudaStream_t s);
void perm_ids_device(const int32_t* perm, const int32_t* in, int32_t* out, int64_t n, cudaStream_t s);
void perm_ids_inplace_device(const int32_t* perm, int32_t* ids, int64_t n, cudaStream_t s);
void perm_ids_valid_device(const int32_t* perm, const int32_t* in, int32_t* out, int64_t n, int64_t nn,
                           cudaStream_t s);
void permute_rows_device(const int32_t* iperm, const double* in, double* out, int64_t nn, int w, bool to_internal,
                         cudaStream_t s);
void permute_rows_u8_device(const int32_t* iperm, const uint8_t* in, uint8_t* out, int64_t nn, bool to_internal,
                            cudaStream_t s);
void export_csr_user_device(const int32_t* perm, const int32_t* iperm, const Pattern& pat, const double* svals,
                            int64_t* uptr, int64_t* udeg, void* scan_tmp, size_t scan_tmp_b, int64_t* row_ptr,
                            int32_t* col_idx, double* vals, cudaStream_t s);
void surface_loads_device(const int64_t* nd_ptr, const int32_t* nd_idx, bool tet, const int32_t* tet_face,
                          const int32_t* face_nodes, const int32_t* face_tet, const uint8_t* flag, const double* xyz,
                          int64_t n_lo, int64_t nloc, const double* t, double* loads, cudaStream_t s);
void apply_bc_device(const int64_t* node_ptr, const int32_t* nbr, const int32_t* diag_slot, int64_t n_lo, int64_t nloc,
                     int64_t nn, const int32_t* dir, int64_t nd, const double* loads, int mode, double penalty_scale,
                     double* vals, double* f, double* dinv, uint8_t* fixed, unsigned long long* flags, cudaStream_t s);

static std::atomic<long long> g_launches{0};
static thread_local bool g_capturing = false;
static thread_local long long g_captured = 0;  // kernels recorded into the graph being captured
void count_launch(long long n) {
  if (!g_capturing) g_launches.fetch_add(n, std::memory_order_relaxed);
  else g_captured += n;
}
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
void set_capturing(bool on) {
  if (on) g_captured = 0;
  g_capturing = on;
}
long long captured_launches() { return g_captured; }

static int g_sms = 0;
int num_sms() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

static long long now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
PhaseTimer::PhaseTimer(cudaStream_t st, const char* tg) : s(st), tag(tg), on(false), t0(0) {
  static const int enabled = [] {
    const char* e = std::getenv("FSFEM_PHASE_TIMES");
    return e != nullptr && e[0] == '1' ? 1 : 0;
  }();
  on = enabled != 0;
  if (on) {
    cudaStreamSynchronize(s);
    t0 = now_ns();
  }
}
void PhaseTimer::mark(const char* name) {
  if (!on) return;
  cudaStreamSynchronize(s);
  const long long t = now_ns();
  std::fprintf(stderr, "  [%s] %-28s %9.3f ms\n", tag, name, (t - t0) * 1e-6);
  t0 = t;
}

// ---- NCCL, resolved at run time (torch has already loaded libnccl.so.2 in practice) ----
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  bool ok = false;
  bool p2p = false;  // send/recv available (halo exchange)
};
static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.p2p = api.Send && api.Recv && api.GroupStart && api.GroupEnd;
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GetErrorString &&
             api.Broadcast && api.GroupStart && api.GroupEnd;
  });
  return api;
}
#define FS_NCCL(call)                                                                                   \
  do {                                                                                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess) throw ::fsfem::Error(FSFEM_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

}  // namespace fsfem

using namespace fsfem;

enum Stage { kCreated = 0, kFaces = 1, kAssembled = 2, kBc = 3 };
// FSFEM_LOOP_AUTO picks the cluster kernel up to this many stored + transposed blocks (measured,
// cfg1, 1.4k blocks: 9.3 vs 15.2 us per iteration; cfg2, 74k: 29 vs 17 us)
constexpr int64_t kClusterAutoBlocks = 8000;

struct fsfem_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int stage = kCreated;
  // partition: rank r owns nodes [ranges[r], ranges[r + 1]) (det.cu: balanced node-face incidences)
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  int64_t n_lo = 0, nloc = 0;
  std::vector<int64_t> ranges{0, 0};
  // loopback group (fsfem_comm_init_loopback): every rank's context in this process, rank order,
  // one device and one stream; collectives become device copies (SURVEY.md §4 simulated partition)
  std::shared_ptr<std::vector<fsfem_ctx*>> loop;
  bool det = false;             // deterministic dots (fsfem_set_deterministic)
  bool overlap = false;         // exchange of the search direction overlapped with the interior SpMV
  cudaStream_t side = nullptr;  // its side stream (created on first use) and fork / join events
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevBuf<double> dpart;         // det: [3 * global chunks] chunk partials
  // mesh
  int64_t nn = 0, nt = 0, nf = 0, ni = 0;
  DevBuf<double> xyz;
  DevBuf<int32_t> tets;
  DevBuf<int32_t> face_nodes, face_tet, face_opp, tet_face;
  DevBuf<int32_t> tet_across;  // [4 nt] vertex across face l of tet t (-1: boundary), for the pattern
  DevBuf<double> xyz_spare;    // spare buffers of the node relabelling (fsfem_set_reorder)
  DevBuf<int32_t> tets_spare, fn_spare, fo_spare;
  // pattern (symmetric block storage, pattern.cuh)
  bool have_pattern = false;
  Pattern pat;
  // numeric
  int method = FSFEM_METHOD_FS;
  double E = 0, nu = 0;
  DevBuf<double> face_s, face_V, vals;  // assembly records (128 B per face / tet) and volumes
  // internal node order (reorder.cu): perm user -> internal, iperm internal -> user
  int reorder_mode = 0;  // 0 auto, 1 always, 2 never
  int pcg_variant = FSFEM_PCG_AUTO;  // requested recurrence (fsfem_set_pcg_variant)
  int exchange = FSFEM_EXCHANGE_ALLGATHER;  // p exchange between ranks (fsfem_set_exchange)
  bool halo_ready = false;                  // send lists agreed with the peers for this pattern
  std::vector<int64_t> halo_need, halo_send;  // per peer: nodes received from / sent to it
  DevBuf<int32_t> halo_send_nodes;          // global ids of own nodes sent, grouped by peer
  DevBuf<double> halo_sbuf, halo_rbuf;      // packed values
  bool cg_active = false;            // recurrence of the current solve / captured graph
  DevBuf<double> cg_p, cg_s;  // single-reduction variant: direction p and s = K p (own rows)
  bool reordered = false;
  double mean_span = 0.0;
  DevBuf<int32_t> perm, iperm, tmp_i;
  DevBuf<double> tmp_d;
  DevBuf<uint8_t> tmp_u8;
  DevBuf<int64_t> exp_tmp;
  DevBuf<unsigned long long> span_tmp;
  // bc / pcg
  DevBuf<double> f, dinv, x_full, r, p_full, q, part, all;
  DevBuf<double> rec_u, rec_strain, rec_stress, rec_nodes, rec_vm;  // stress recovery
  DevBuf<uint8_t> fixed;
  DevBuf<PcgState> st;
  DevBuf<unsigned char> scratch;
  DevBuf<unsigned long long> flags;
  DevBuf<double> staging;  // host->device staging for loads / u
  DevBuf<int32_t> staging_i;
  unsigned long long* h_flags = nullptr;  // pinned [8]
  PcgState* h_st = nullptr;               // pinned
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> spmv_ev;
  fsfem_report rep{};
  // graph cache: every pointer and size the captured iterations bake in (graph_key_of)
  cudaGraphExec_t graph = nullptr;
  std::vector<uintptr_t> graph_key;
  long long graph_launches = 0;  // kernels per replay of the graph (counted at capture)
  // device-side loop (default): one graph whose while node repeats a body of kDevBatch iterations
  // until the recurrence stops -- no host synchronisation inside the solve
  int loop_mode = FSFEM_LOOP_AUTO;  // cluster kernel for small meshes, else host batches
  DevBuf<int64_t> cl_split;         // row split of the cluster PCG kernel
  cudaGraphExec_t dgraph = nullptr;
  std::vector<uintptr_t> dgraph_key;
  long long dgraph_body_launches = 0;
  bool dgraph_failed = false;  // instantiation refused (e.g. collectives inside the body): host batches
  int max_restarts = 2;  // residual-replacement restarts when the true residual misses (fsfem_pcg_solve)
};

namespace {

constexpr int kBatch = 32;     // PCG iterations per CUDA graph launch (host-polled loop)
constexpr int kDevBatch = 8;   // PCG iterations per body of the device-side while loop

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Copy `bytes` from a host-or-device source into device memory dst (stream ordered).
void to_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  FS_CUDA(cudaMemcpyAsync(dst, src, bytes, is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
}
void from_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0 || !dst) return;
  FS_CUDA(cudaMemcpyAsync(dst, src, bytes, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
}

template <typename T>
void swap_buf(DevBuf<T>& a, DevBuf<T>& b) {
  std::swap(a.p, b.p);
  std::swap(a.n, b.n);
}

// Node-indexed input (nn rows of w doubles, caller's numbering, host or device) -> device, internal
// numbering.  Uses c->staging (must hold w*nn) when a permutation is needed.
const double* node_in(fsfem_ctx* c, const double* user, int w, double* dst);
// Device internal-numbered rows -> caller's array (host or device), caller's numbering.
void node_out(fsfem_ctx* c, double* user, const double* internal, int64_t row0, int64_t nrows, int w);

fsfem_status fail(fsfem_ctx* c, fsfem_status code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

template <typename F>
fsfem_status guarded(fsfem_ctx* c, F&& fn) {
  if (!c) return FSFEM_ERR_INVALID_ARG;
  try {
    c->err.clear();
    FS_CUDA(cudaSetDevice(c->device));
    return fn();
  } catch (const Error& e) {
    c->err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failed";
    return FSFEM_ERR_OOM;
  } catch (const std::exception& e) {
    c->err = e.what();
    return FSFEM_ERR_CUDA;
  }
}

fsfem_status decode_flags(fsfem_ctx* c, unsigned long long v, const char* what) {
  if (v == kNoError) return FSFEM_OK;
  const int code = static_cast<int>(v >> 56);
  const long long idx = static_cast<long long>(v & ((1ull << 56) - 1));
  const char* item = "item";
  switch (code) {
    case FSFEM_ERR_INVALID_ARG: item = "entry"; break;
    case FSFEM_ERR_DEGENERATE: item = "tet"; break;
    case FSFEM_ERR_TOPOLOGY: item = "face bucket (smallest node id)"; break;
    case FSFEM_ERR_UNSUPPORTED: item = "node"; break;
    case FSFEM_ERR_BREAKDOWN: item = "dof"; break;
    default: break;
  }
  c->err = std::string(what) + ": " + fsfem_status_string(static_cast<fsfem_status>(code)) + " at " + item + " " +
           std::to_string(idx);
  return static_cast<fsfem_status>(code);
}

const double* node_in(fsfem_ctx* c, const double* user, int w, double* dst) {
  if (!c->reordered) {
    to_device(dst, user, sizeof(double) * w * c->nn, c->stream);
    return dst;
  }
  double* tmp = c->tmp_d.ensure(static_cast<size_t>(w) * c->nn);
  to_device(tmp, user, sizeof(double) * w * c->nn, c->stream);
  permute_rows_device(c->iperm.get(), tmp, dst, c->nn, w, true, c->stream);
  return dst;
}

void node_out(fsfem_ctx* c, double* user, const double* internal, int64_t row0, int64_t nrows, int w) {
  if (!user || nrows <= 0) return;
  if (!c->reordered) {
    from_device(user + static_cast<int64_t>(w) * row0, internal, sizeof(double) * w * nrows, c->stream);
    return;
  }
  double* tmp = c->tmp_d.ensure(static_cast<size_t>(w) * c->nn);  // single rank: row0 = 0, nrows = nn
  permute_rows_device(c->iperm.get(), internal, tmp, c->nn, w, false, c->stream);
  from_device(user, tmp, sizeof(double) * w * c->nn, c->stream);
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  FS_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

void drop_graph(fsfem_ctx* c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  c->graph = nullptr;
  c->graph_key.clear();
  if (c->dgraph) cudaGraphExecDestroy(c->dgraph);
  c->dgraph = nullptr;
  c->dgraph_key.clear();
}

// ---- collectives over the ranks of one solve ---------------------------------------------------
// `cs` holds the contexts this process drives: {c} with NCCL (one rank per process), or every
// rank's context with the loopback group.  The per-rank kernels are the same in both cases;
// only the data movement of a collective differs (NCCL calls vs device-to-device copies on the
// shared stream), so the loopback group executes the multi-rank code path on one GPU.
using Ranks = std::vector<fsfem_ctx*>;

Ranks ranks_of(fsfem_ctx* c) { return c->loop ? *c->loop : Ranks{c}; }

void d2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes) FS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
}

// Every rank's 4 partials (st->local) into every rank's `all` (rank order), then the combine step.
void coll_partials(const Ranks& cs, int stage) {
  fsfem_ctx* c0 = cs[0];
  if (c0->nranks == 1) return;
  if (c0->loop) {
    for (fsfem_ctx* d : cs)
      for (fsfem_ctx* q : cs) d2d(d->all.get() + 4 * q->rank, q->st.get()->local, 4 * sizeof(double), d->stream);
  } else {
    FS_NCCL(nccl().AllGather(c0->st.get()->local, c0->all.get(), 4, ncclDouble, c0->comm, c0->stream));
  }
  for (fsfem_ctx* c : cs) launch_combine(c->st.get(), c->all.get(), stage, c->nranks, c->stream);
}

// All-gather (v) of the own node-range slices of a full-length vector (3 doubles per node).
void coll_allgatherv(const Ranks& cs, DevBuf<double> fsfem_ctx::*buf) {
  fsfem_ctx* c0 = cs[0];
  if (c0->nranks == 1) return;
  const std::vector<int64_t>& R = c0->ranges;
  if (c0->loop) {
    for (fsfem_ctx* q : cs) {
      const int64_t lo = R[q->rank], n = R[q->rank + 1] - lo;
      for (fsfem_ctx* d : cs)
        if (d != q) d2d((d->*buf).get() + 3 * lo, (q->*buf).get() + 3 * lo, sizeof(double) * 3 * n, d->stream);
    }
    return;
  }
  double* full = (c0->*buf).get();
  FS_NCCL(nccl().GroupStart());
  for (int q = 0; q < c0->nranks; ++q) {
    const int64_t lo = R[q], n = R[q + 1] - lo;
    if (n > 0) FS_NCCL(nccl().Broadcast(full + 3 * lo, full + 3 * lo, 3 * n, ncclDouble, q, c0->comm, c0->stream));
  }
  FS_NCCL(nccl().GroupEnd());
}

// Halo mode: each rank receives only the entries of its halo (halo.cu) from their owners and
// sends the entries its peers need; the other remote entries of the vector are left stale (the
// SpMV never reads them).  Fixed send/recv sizes per peer, agreed once per pattern (setup_halo).
void coll_halo(const Ranks& cs, DevBuf<double> fsfem_ctx::*buf) {
  for (fsfem_ctx* c : cs) {
    int64_t ns = 0;
    for (int q = 0; q < c->nranks; ++q) ns += c->halo_send[q];
    halo_pack_device((c->*buf).get(), c->halo_send_nodes.get(), ns, c->halo_sbuf.get(), c->stream);
  }
  fsfem_ctx* c0 = cs[0];
  const int nr = c0->nranks;
  if (c0->loop) {
    for (fsfem_ctx* q : cs) {  // sender q -> receiver d
      int64_t so = 0;
      for (fsfem_ctx* d : cs) {
        const int64_t n = q->halo_send[d->rank];
        int64_t ro = 0;
        for (int k = 0; k < q->rank; ++k) ro += d->halo_need[k];
        if (d != q) d2d(d->halo_rbuf.get() + 3 * ro, q->halo_sbuf.get() + 3 * so, sizeof(double) * 3 * n, d->stream);
        so += n;
      }
    }
  } else {
    FS_NCCL(nccl().GroupStart());
    int64_t so = 0, ro = 0;
    for (int q = 0; q < nr; ++q) {
      if (c0->halo_send[q] > 0)
        FS_NCCL(nccl().Send(c0->halo_sbuf.get() + 3 * so, 3 * c0->halo_send[q], ncclDouble, q, c0->comm, c0->stream));
      if (c0->halo_need[q] > 0)
        FS_NCCL(nccl().Recv(c0->halo_rbuf.get() + 3 * ro, 3 * c0->halo_need[q], ncclDouble, q, c0->comm, c0->stream));
      so += c0->halo_send[q];
      ro += c0->halo_need[q];
    }
    FS_NCCL(nccl().GroupEnd());
  }
  for (fsfem_ctx* c : cs) halo_unpack_device(c->halo_rbuf.get(), c->pat.halo.get(), c->pat.nhalo, (c->*buf).get(), c->stream);
}

// The search direction (p, or u in the single-reduction form) before an SpMV.
void coll_full(const Ranks& cs, DevBuf<double> fsfem_ctx::*buf) {
  if (cs[0]->nranks == 1) return;
  if (cs[0]->exchange == FSFEM_EXCHANGE_HALO) coll_halo(cs, buf);
  else coll_allgatherv(cs, buf);
}

// Deterministic mode: the chunk partials of every rank's chunk range to every rank.
void coll_dpart(const Ranks& cs) {
  fsfem_ctx* c0 = cs[0];
  if (c0->nranks == 1) return;
  const std::vector<int64_t>& R = c0->ranges;
  auto crange = [&](int q, int64_t& a, int64_t& n) {
    a = R[q] / kDetChunkNodes;
    n = ceil_div(R[q + 1], kDetChunkNodes) - a;
    if (R[q + 1] <= R[q]) n = 0;
  };
  if (c0->loop) {
    for (fsfem_ctx* q : cs) {
      int64_t a, n;
      crange(q->rank, a, n);
      for (fsfem_ctx* d : cs)
        if (d != q) d2d(d->dpart.get() + 3 * a, q->dpart.get() + 3 * a, sizeof(double) * 3 * n, d->stream);
    }
    return;
  }
  FS_NCCL(nccl().GroupStart());
  for (int q = 0; q < c0->nranks; ++q) {
    int64_t a, n;
    crange(q, a, n);
    if (n > 0)
      FS_NCCL(nccl().Broadcast(c0->dpart.get() + 3 * a, c0->dpart.get() + 3 * a, 3 * n, ncclDouble, q, c0->comm,
                               c0->stream));
  }
  FS_NCCL(nccl().GroupEnd());
}

// Agree on the halo exchange (once per pattern): every rank learns from each owner how many of
// the owner's nodes it needs and sends it the list (NCCL: all-gather of the counts, send/recv of
// the lists; loopback: read directly from the peers' contexts).
void setup_halo(const Ranks& cs) {
  fsfem_ctx* c0 = cs[0];
  const int nr = c0->nranks;
  if (c0->loop) {
    for (fsfem_ctx* q : cs) {  // q sends to d what d needs from q: a slice of d's halo (grouped by owner)
      q->halo_send.assign(nr, 0);
      int64_t ns = 0;
      for (fsfem_ctx* d : cs) {
        q->halo_send[d->rank] = d == q ? 0 : d->halo_need[q->rank];
        ns += q->halo_send[d->rank];
      }
      q->halo_send_nodes.ensure(std::max<int64_t>(ns, 1));
      q->halo_sbuf.ensure(3 * std::max<int64_t>(ns, 1));
      int64_t so = 0;
      for (fsfem_ctx* d : cs) {
        int64_t off = 0;
        for (int k = 0; k < q->rank; ++k) off += d->halo_need[k];
        d2d(q->halo_send_nodes.get() + so, d->pat.halo.get() + off, sizeof(int32_t) * q->halo_send[d->rank], q->stream);
        so += q->halo_send[d->rank];
      }
      int64_t nneed = 0;
      for (int k = 0; k < nr; ++k) nneed += q->halo_need[k];
      q->halo_rbuf.ensure(3 * std::max<int64_t>(nneed, 1));
    }
    FS_CUDA(cudaStreamSynchronize(c0->stream));
    for (fsfem_ctx* q : cs) q->halo_ready = true;
    return;
  }
  fsfem_ctx* c = c0;
  const int me = c->rank;
  if (!nccl().p2p) throw Error(FSFEM_ERR_NCCL, "ncclSend/ncclRecv not available for the halo exchange");
  DevBuf<int64_t> cnt, all;
  cnt.ensure(nr);
  all.ensure(static_cast<size_t>(nr) * nr);
  FS_CUDA(cudaMemcpyAsync(cnt.get(), c->halo_need.data(), sizeof(int64_t) * nr, cudaMemcpyHostToDevice, c->stream));
  FS_NCCL(nccl().AllGather(cnt.get(), all.get(), nr, ncclInt64, c->comm, c->stream));
  std::vector<int64_t> h(static_cast<size_t>(nr) * nr);
  FS_CUDA(cudaMemcpyAsync(h.data(), all.get(), sizeof(int64_t) * nr * nr, cudaMemcpyDeviceToHost, c->stream));
  FS_CUDA(cudaStreamSynchronize(c->stream));
  c->halo_send.assign(nr, 0);
  int64_t ns = 0, nneed = 0;
  for (int q = 0; q < nr; ++q) {
    c->halo_send[q] = q == me ? 0 : h[static_cast<size_t>(q) * nr + me];  // what q needs from me
    ns += c->halo_send[q];
    nneed += c->halo_need[q];
  }
  c->halo_send_nodes.ensure(std::max<int64_t>(ns, 1));
  c->halo_sbuf.ensure(3 * std::max<int64_t>(ns, 1));
  c->halo_rbuf.ensure(3 * std::max<int64_t>(nneed, 1));
  FS_NCCL(nccl().GroupStart());
  int64_t so = 0, ro = 0;
  for (int q = 0; q < nr; ++q) {
    if (c->halo_need[q] > 0)
      FS_NCCL(nccl().Send(c->pat.halo.get() + ro, c->halo_need[q], ncclInt32, q, c->comm, c->stream));
    if (c->halo_send[q] > 0)
      FS_NCCL(nccl().Recv(c->halo_send_nodes.get() + so, c->halo_send[q], ncclInt32, q, c->comm, c->stream));
    so += c->halo_send[q];
    ro += c->halo_need[q];
  }
  FS_NCCL(nccl().GroupEnd());
  FS_CUDA(cudaStreamSynchronize(c->stream));
  c->halo_ready = true;
}

// Overlap: the exchange of the search direction runs on a side stream while the
// interior chunks (no column outside the rank's range) are multiplied; the boundary chunks follow
// once the exchange has landed.  Fork / join by events, so it is captured into the graphs too.
bool overlapping(const Ranks& cs) {
  const fsfem_ctx* c0 = cs[0];
  return c0->overlap && c0->nranks > 1 && !c0->det;
}

void spmv_with_exchange(const Ranks& cs, DevBuf<double> fsfem_ctx::*buf, DevBuf<double> fsfem_ctx::*out,
                        cudaEvent_t e0, cudaEvent_t e1) {
  fsfem_ctx* c0 = cs[0];
  if (!c0->side) {
    FS_CUDA(cudaStreamCreateWithFlags(&c0->side, cudaStreamNonBlocking));
    FS_CUDA(cudaEventCreateWithFlags(&c0->ev_fork, cudaEventDisableTiming));
    FS_CUDA(cudaEventCreateWithFlags(&c0->ev_join, cudaEventDisableTiming));
  }
  cudaStream_t main = c0->stream;
  FS_CUDA(cudaEventRecord(c0->ev_fork, main));
  FS_CUDA(cudaStreamWaitEvent(c0->side, c0->ev_fork, 0));
  std::vector<cudaStream_t> saved;
  for (fsfem_ctx* c : cs) {  // the collective code path, issued on the side stream
    saved.push_back(c->stream);
    c->stream = c0->side;
  }
  try {
    coll_full(cs, buf);
  } catch (...) {
    for (size_t k = 0; k < cs.size(); ++k) cs[k]->stream = saved[k];
    throw;
  }
  for (size_t k = 0; k < cs.size(); ++k) cs[k]->stream = saved[k];
  FS_CUDA(cudaEventRecord(c0->ev_join, c0->side));
  for (fsfem_ctx* c : cs) {
    if (e0 && c == c0) FS_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
    launch_spmv_split(c->pat, 1, c->vals.get(), (c->*buf).get(), 3 * c->n_lo, (c->*out).get(), c->st.get(),
                      c->part.get(), c->stream);
  }
  FS_CUDA(cudaStreamWaitEvent(main, c0->ev_join, 0));
  for (fsfem_ctx* c : cs) {
    launch_spmv_split(c->pat, 2, c->vals.get(), (c->*buf).get(), 3 * c->n_lo, (c->*out).get(), c->st.get(),
                      c->part.get(), c->stream);
    if (e1 && c == c0) FS_CUDA(cudaEventRecordWithFlags(e1, c->stream, cudaEventRecordExternal));
  }
}

// ---- one PCG iteration over the ranks ----------------------------------------------------------
double* own_p(fsfem_ctx* c) { return c->p_full.get() + 3 * c->n_lo; }
double* own_x(fsfem_ctx* c) { return c->x_full.get() + 3 * c->n_lo; }

void spmv_of(fsfem_ctx* c, const double* x_full, double* y, bool pcg) {
  if (c->det) launch_spmv_canon(c->pat, c->vals.get(), x_full, y, pcg ? c->st.get() : nullptr, c->stream);
  else launch_spmv(c->pat, c->vals.get(), x_full, 3 * c->n_lo, y, pcg ? c->st.get() : nullptr, c->part.get(), pcg,
                   c->stream);
}

// Single-reduction iteration (Chronopoulos-Gear): update (x, r, u = D^-1 r,
// p, s; partials of r.u and r.r), exchange of u, SpMV w = K u with u.w, and ONE combined
// reduction (u.w, r.u, r.r) -> alpha, beta.  p_full holds u, q holds w.
void iter_cg(const Ranks& cs, cudaEvent_t e0, cudaEvent_t e1) {
  for (fsfem_ctx* c : cs)
    launch_cg_update(own_x(c), c->r.get(), own_p(c), c->cg_p.get(), c->cg_s.get(), c->q.get(), c->dinv.get(),
                     3 * c->nloc, c->st.get(), c->part.get() + 4 * pcg_grid(), c->stream);
  if (overlapping(cs)) {
    spmv_with_exchange(cs, &fsfem_ctx::p_full, &fsfem_ctx::q, e0, e1);
  } else {
    coll_full(cs, &fsfem_ctx::p_full);
    for (fsfem_ctx* c : cs) {
      if (e0 && c == cs[0]) FS_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
      spmv_of(c, c->p_full.get(), c->q.get(), true);
      if (e1 && c == cs[0]) FS_CUDA(cudaEventRecordWithFlags(e1, c->stream, cudaEventRecordExternal));
    }
  }
  coll_partials(cs, 4);
}

// Deterministic dots (det.cu): SpMV in canonical order, chunk partials of p.q, exchange, sum in
// chunk order -> alpha; update with chunk partials of r.r, r.z, exchange -> beta; direction.
void iter_det(const Ranks& cs, cudaEvent_t e0, cudaEvent_t e1) {
  for (fsfem_ctx* c : cs) {
    if (e0 && c == cs[0]) FS_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
    spmv_of(c, c->p_full.get(), c->q.get(), true);
    if (e1 && c == cs[0]) FS_CUDA(cudaEventRecordWithFlags(e1, c->stream, cudaEventRecordExternal));
    launch_det_dots(1, c->n_lo, c->nloc, nullptr, c->q.get(), nullptr, nullptr, own_p(c), nullptr, c->st.get(),
                    c->dpart.get(), c->stream);
  }
  coll_dpart(cs);
  for (fsfem_ctx* c : cs) {
    launch_det_finish(c->st.get(), c->dpart.get(), det_nchunks(c->nn), 1, c->stream);
    launch_det_dots(2, c->n_lo, c->nloc, nullptr, c->q.get(), c->dinv.get(), c->r.get(), own_p(c), own_x(c),
                    c->st.get(), c->dpart.get(), c->stream);
  }
  coll_dpart(cs);
  for (fsfem_ctx* c : cs) {
    launch_det_finish(c->st.get(), c->dpart.get(), det_nchunks(c->nn), 2, c->stream);
    launch_direction(own_p(c), c->r.get(), c->dinv.get(), 3 * c->nloc, c->st.get(), c->stream);
  }
  coll_full(cs, &fsfem_ctx::p_full);
}

void pcg_iteration(const Ranks& cs, cudaEvent_t e0, cudaEvent_t e1) {
  fsfem_ctx* c0 = cs[0];
  if (c0->det) return iter_det(cs, e0, e1);
  if (c0->cg_active) return iter_cg(cs, e0, e1);
  const bool ov = overlapping(cs);
  if (ov) {  // this iteration's exchange of p (issued at its start, see below) overlaps the interior rows
    spmv_with_exchange(cs, &fsfem_ctx::p_full, &fsfem_ctx::q, e0, e1);
  } else {
    for (fsfem_ctx* c : cs) {
      if (e0 && c == c0) FS_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
      spmv_of(c, c->p_full.get(), c->q.get(), true);
      if (e1 && c == c0) FS_CUDA(cudaEventRecordWithFlags(e1, c->stream, cudaEventRecordExternal));
    }
  }
  if (c0->nranks == 1) {
    launch_update_direction(own_x(c0), c0->r.get(), own_p(c0), c0->q.get(), c0->dinv.get(), 3 * c0->nloc,
                            c0->st.get(), c0->part.get(), c0->stream);
    return;
  }
  coll_partials(cs, 1);
  for (fsfem_ctx* c : cs)
    launch_update(own_x(c), c->r.get(), own_p(c), c->q.get(), c->dinv.get(), 3 * c->nloc, c->st.get(), c->part.get(),
                  c->stream);
  coll_partials(cs, 2);
  for (fsfem_ctx* c : cs) launch_direction(own_p(c), c->r.get(), c->dinv.get(), 3 * c->nloc, c->st.get(), c->stream);
  if (!ov) coll_full(cs, &fsfem_ctx::p_full);  // (overlap: exchanged at the next SpMV)
}

// Everything a captured batch of iterations bakes in: buffer pointers of every rank, sizes,
// halo counts, variant and mode.  A graph is replayed only while its key is unchanged.
std::vector<uintptr_t> graph_key_of(const Ranks& cs) {
  std::vector<uintptr_t> k;
  auto P = [&](const void* p) { k.push_back(reinterpret_cast<uintptr_t>(p)); };
  for (fsfem_ctx* c : cs) {
    P(c);
    P(c->stream);
    P(c->vals.get());
    P(c->x_full.get());
    P(c->p_full.get());
    P(c->r.get());
    P(c->q.get());
    P(c->f.get());
    P(c->dinv.get());
    P(c->part.get());
    P(c->all.get());
    P(c->st.get());
    P(c->cg_p.get());
    P(c->cg_s.get());
    P(c->dpart.get());
    P(c->halo_sbuf.get());
    P(c->halo_rbuf.get());
    P(c->halo_send_nodes.get());
    P(c->pat.halo.get());
    P(c->pat.sptr.get());
    P(c->pat.tbuf.get());
    k.push_back(static_cast<uintptr_t>(c->n_lo));
    k.push_back(static_cast<uintptr_t>(c->nloc));
    k.push_back(static_cast<uintptr_t>(c->nranks));
    k.push_back(static_cast<uintptr_t>(c->exchange));
    k.push_back(static_cast<uintptr_t>(c->cg_active));
    k.push_back(static_cast<uintptr_t>(c->det));
    k.push_back(static_cast<uintptr_t>(c->overlap));
    for (int64_t v : c->halo_send) k.push_back(static_cast<uintptr_t>(v));
    for (int64_t v : c->halo_need) k.push_back(static_cast<uintptr_t>(v));
    for (int64_t v : c->ranges) k.push_back(static_cast<uintptr_t>(v));
  }
  return k;
}

}  // namespace

extern "C" {

const char* fsfem_status_string(fsfem_status s) {
  switch (s) {
    case FSFEM_OK: return "ok";
    case FSFEM_ERR_INVALID_ARG: return "invalid argument";
    case FSFEM_ERR_TOPOLOGY: return "topology error";
    case FSFEM_ERR_DEGENERATE: return "degenerate element";
    case FSFEM_ERR_UNSUPPORTED: return "unsupported size";
    case FSFEM_ERR_NOT_CONVERGED: return "not converged";
    case FSFEM_ERR_BREAKDOWN: return "breakdown";
    case FSFEM_ERR_STATE: return "call order violated";
    case FSFEM_ERR_CUDA: return "cuda error";
    case FSFEM_ERR_NCCL: return "nccl error";
    case FSFEM_ERR_OOM: return "out of device memory";
  }
  return "unknown status";
}

fsfem_status fsfem_create(int cuda_device, void* cuda_stream, fsfem_ctx** out) {
  if (!out) return FSFEM_ERR_INVALID_ARG;
  *out = nullptr;
  fsfem_ctx* c = new (std::nothrow) fsfem_ctx();
  if (!c) return FSFEM_ERR_OOM;
  c->device = cuda_device;
  fsfem_status st = guarded(c, [&]() -> fsfem_status {
    if (cuda_stream) {
      c->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
      FS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    FS_CUDA(cudaMallocHost(&c->h_flags, 8 * sizeof(unsigned long long)));
    FS_CUDA(cudaMallocHost(&c->h_st, sizeof(PcgState)));
    FS_CUDA(cudaEventCreate(&c->ev0));
    FS_CUDA(cudaEventCreate(&c->ev1));
    c->spmv_ev.resize(2 * kBatch);
    for (auto& e : c->spmv_ev) FS_CUDA(cudaEventCreate(&e));
    c->flags.ensure(8);
    c->st.ensure(1);
    num_sms();
    return FSFEM_OK;
  });
  if (st != FSFEM_OK) {
    fsfem_destroy(c);
    return st;
  }
  *out = c;
  return FSFEM_OK;
}

fsfem_status fsfem_destroy(fsfem_ctx* c) {
  if (!c) return FSFEM_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graph(c);
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (auto e : c->spmv_ev)
    if (e) cudaEventDestroy(e);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  if (c->h_st) cudaFreeHost(c->h_st);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return FSFEM_OK;
}

const char* fsfem_last_error(const fsfem_ctx* c) { return c ? c->err.c_str() : "null context"; }

fsfem_status fsfem_nccl_get_unique_id(void* out) {
  if (!out) return FSFEM_ERR_INVALID_ARG;
  if (!nccl().ok) return FSFEM_ERR_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return FSFEM_ERR_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return FSFEM_OK;
}

fsfem_status fsfem_comm_init(fsfem_ctx* c, const void* uid, int rank, int nranks) {
  return guarded(c, [&]() -> fsfem_status {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, FSFEM_ERR_INVALID_ARG, "bad rank/nranks");
    if (c->stage != kCreated) return fail(c, FSFEM_ERR_STATE, "comm_init must precede build_faces");
    if (nranks > 1 && uid) {
      if (!nccl().ok) return fail(c, FSFEM_ERR_NCCL, "libnccl.so.2 not loadable");
      ncclUniqueId id;
      std::memcpy(&id, uid, sizeof(id));
      FS_NCCL(nccl().CommInitRank(&c->comm, nranks, id, rank));
    }
    c->rank = rank;
    c->nranks = nranks;
    c->loop.reset();
    return FSFEM_OK;
  });
}

fsfem_status fsfem_comm_init_loopback(fsfem_ctx** ctxs, int nranks) {
  if (!ctxs || nranks < 1) return FSFEM_ERR_INVALID_ARG;
  for (int r = 0; r < nranks; ++r)
    if (!ctxs[r]) return FSFEM_ERR_INVALID_ARG;
  for (int r = 0; r < nranks; ++r)
    for (int q = 0; q < r; ++q)
      if (ctxs[q] == ctxs[r]) return fail(ctxs[0], FSFEM_ERR_INVALID_ARG, "the contexts of a loopback group must be distinct");
  for (int r = 0; r < nranks; ++r) {
    fsfem_ctx* c = ctxs[r];
    if (c->stage != kCreated) return fail(ctxs[0], FSFEM_ERR_STATE, "comm_init_loopback must precede build_faces");
    if (c->device != ctxs[0]->device || c->stream != ctxs[0]->stream)
      return fail(ctxs[0], FSFEM_ERR_INVALID_ARG, "a loopback group shares one device and one stream");
    if (c->comm) return fail(ctxs[0], FSFEM_ERR_STATE, "context already joined an NCCL communicator");
  }
  auto group = std::make_shared<std::vector<fsfem_ctx*>>(ctxs, ctxs + nranks);
  for (int r = 0; r < nranks; ++r) {
    ctxs[r]->rank = r;
    ctxs[r]->nranks = nranks;
    ctxs[r]->loop = group;
  }
  return FSFEM_OK;
}

fsfem_status fsfem_set_overlap(fsfem_ctx* c, int on) {
  return guarded(c, [&]() -> fsfem_status {
    c->overlap = on != 0;
    return FSFEM_OK;
  });
}

fsfem_status fsfem_set_loop(fsfem_ctx* c, int mode) {
  return guarded(c, [&]() -> fsfem_status {
    if (mode < FSFEM_LOOP_DEVICE || mode > FSFEM_LOOP_AUTO)
      return fail(c, FSFEM_ERR_INVALID_ARG, "loop mode must be 0 (device), 1 (host), 2 (cluster) or 3 (auto)");
    c->loop_mode = mode;
    return FSFEM_OK;
  });
}

fsfem_status fsfem_set_deterministic(fsfem_ctx* c, int on) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage != kCreated) return fail(c, FSFEM_ERR_STATE, "set_deterministic must precede build_faces");
    c->det = on != 0;
    drop_graph(c);
    return FSFEM_OK;
  });
}

fsfem_status fsfem_get_partition(const fsfem_ctx* cc, int64_t* ranges) {
  fsfem_ctx* c = const_cast<fsfem_ctx*>(cc);
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kFaces) return fail(c, FSFEM_ERR_STATE, "build_faces first");
    if (!ranges) return fail(c, FSFEM_ERR_INVALID_ARG, "null ranges");
    for (int r = 0; r <= c->nranks; ++r) ranges[r] = c->ranges[r];
    return FSFEM_OK;
  });
}

fsfem_status fsfem_set_method(fsfem_ctx* c, int method) {
  return guarded(c, [&]() -> fsfem_status {
    if (method != FSFEM_METHOD_FS && method != FSFEM_METHOD_FEM_T4)
      return fail(c, FSFEM_ERR_INVALID_ARG, "method must be FSFEM_METHOD_FS or FSFEM_METHOD_FEM_T4");
    if (method != c->method) {
      c->method = method;
      c->have_pattern = false;  // different node graph
      drop_graph(c);
      if (c->stage > kFaces) c->stage = kFaces;
    }
    return FSFEM_OK;
  });
}

fsfem_status fsfem_set_exchange(fsfem_ctx* c, int mode) {
  return guarded(c, [&]() -> fsfem_status {
    if (mode != FSFEM_EXCHANGE_ALLGATHER && mode != FSFEM_EXCHANGE_HALO)
      return fail(c, FSFEM_ERR_INVALID_ARG, "exchange must be 0 (all-gather) or 1 (halo)");
    if (c->stage >= kAssembled && mode != c->exchange)
      return fail(c, FSFEM_ERR_STATE, "set the exchange before the first assemble_csr of a mesh");
    c->exchange = mode;
    return FSFEM_OK;
  });
}

fsfem_status fsfem_get_halo(const fsfem_ctx* cc, int32_t* nodes, int64_t* n) {
  fsfem_ctx* c = const_cast<fsfem_ctx*>(cc);
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kAssembled) return fail(c, FSFEM_ERR_STATE, "assemble_csr first");
    const int64_t nh = c->nranks > 1 ? c->pat.nhalo : 0;
    if (n) *n = nh;
    if (nodes && nh > 0) from_device(nodes, c->pat.halo.get(), sizeof(int32_t) * nh, c->stream);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_set_pcg_variant(fsfem_ctx* c, int variant) {
  return guarded(c, [&]() -> fsfem_status {
    if (variant != FSFEM_PCG_STANDARD && variant != FSFEM_PCG_SINGLE_REDUCTION && variant != FSFEM_PCG_AUTO)
      return fail(c, FSFEM_ERR_INVALID_ARG, "pcg variant must be 0 (standard), 1 (single reduction) or 2 (auto)");
    if (variant != c->pcg_variant) drop_graph(c);
    c->pcg_variant = variant;
    return FSFEM_OK;
  });
}

fsfem_status fsfem_set_reorder(fsfem_ctx* c, int mode) {
  return guarded(c, [&]() -> fsfem_status {
    if (mode < 0 || mode > 2) return fail(c, FSFEM_ERR_INVALID_ARG, "reorder mode must be 0 (auto), 1 (always) or 2 (never)");
    c->reorder_mode = mode;  // takes effect at the next fsfem_build_faces
    return FSFEM_OK;
  });
}

fsfem_status fsfem_build_faces(fsfem_ctx* c, const double* xyz, int64_t n_nodes, const int32_t* tets, int64_t n_tets,
                               int64_t* n_faces, int64_t* n_interior) {
  return guarded(c, [&]() -> fsfem_status {
    if (!xyz || !tets || n_nodes < 4 || n_tets < 1) return fail(c, FSFEM_ERR_INVALID_ARG, "need >= 4 nodes and >= 1 tet");
    if (n_nodes >= (1LL << 31) / 3 || 4 * n_tets >= (1LL << 31))
      return fail(c, FSFEM_ERR_UNSUPPORTED, "mesh too large for 32-bit ids");
    drop_graph(c);
    c->stage = kCreated;
    c->have_pattern = false;
    c->halo_ready = false;
    c->nn = n_nodes;
    c->nt = n_tets;
    c->xyz.ensure(3 * n_nodes);
    c->tets.ensure(4 * n_tets);
    FS_CUDA(cudaEventRecord(c->ev0, c->stream));
    to_device(c->xyz.get(), xyz, sizeof(double) * 3 * n_nodes, c->stream);
    to_device(c->tets.get(), tets, sizeof(int32_t) * 4 * n_tets, c->stream);
    int64_t nf = 0, ni = 0;
    c->h_flags[0] = kNoError;
    build_faces_device(c->xyz.get(), n_nodes, c->tets.get(), n_tets, c->stream, c->scratch, c->face_nodes, c->face_tet,
                       c->face_opp, c->tet_face, c->tet_across, &nf, &ni, c->h_flags);
    fsfem_status s = decode_flags(c, c->h_flags[0], "build_faces");
    if (s != FSFEM_OK) return s;
    PhaseTimer pt(c->stream, "faces");
    // row partition: node ranges balanced by node-face incidences, aligned to
    // the deterministic dot chunk when that mode is on (every rank computes the same ranges)
    partition_ranges_device(c->face_nodes.get(), c->face_opp.get(), nf, n_nodes, c->nranks, c->det ? kDetChunkNodes : 32,
                            c->scratch, c->stream, c->ranges);
    c->n_lo = c->ranges[c->rank];
    c->nloc = c->ranges[c->rank + 1] - c->n_lo;
    // Internal node order (reorder.cu): renumber in Morton order when the caller's numbering is
    // not banded (mean tet id span > 16 N^(2/3)), never with several ranks (the documented row
    // partition is in the caller's numbering).
    pt.mark("partition ranges");
    c->span_tmp.ensure(1);
    c->mean_span = mean_tet_span_device(c->tets.get(), n_tets, c->span_tmp.get(), c->stream);
    pt.mark("mean tet span");
    const bool want = c->nranks == 1 &&
                      (c->reorder_mode == 1 ||
                       (c->reorder_mode == 0 && c->mean_span > 16.0 * std::pow(static_cast<double>(n_nodes), 2.0 / 3.0)));
    c->reordered = false;
    if (want) {
      c->iperm.ensure(n_nodes);
      c->perm.ensure(n_nodes);
      morton_order_device(c->xyz.get(), n_nodes, c->iperm.get(), c->perm.get(), c->scratch, c->stream);
      // the matrix path works on the renumbered mesh; faces keep their ids and order
      // the relabelled copies go to persistent spare buffers (swapped in; the old arrays become the
      // spares of the next call): no cudaMalloc / cudaFree of ~0.6 GB per call at cfg5
      DevBuf<double>& xyz_i = c->xyz_spare;
      xyz_i.ensure(3 * n_nodes);
      permute_rows_device(c->iperm.get(), c->xyz.get(), xyz_i.get(), n_nodes, 3, true, c->stream);
      DevBuf<int32_t>& tets_i = c->tets_spare;
      DevBuf<int32_t>& fn_i = c->fn_spare;
      DevBuf<int32_t>& fo_i = c->fo_spare;
      tets_i.ensure(4 * n_tets);
      fn_i.ensure(3 * nf);
      fo_i.ensure(2 * nf);
      perm_ids_device(c->perm.get(), c->tets.get(), tets_i.get(), 4 * n_tets, c->stream);
      perm_ids_device(c->perm.get(), c->face_nodes.get(), fn_i.get(), 3 * nf, c->stream);
      perm_ids_device(c->perm.get(), c->face_opp.get(), fo_i.get(), 2 * nf, c->stream);
      perm_ids_inplace_device(c->perm.get(), c->tet_across.get(), 4 * n_tets, c->stream);  // no temporary
      FS_CUDA(cudaStreamSynchronize(c->stream));
      swap_buf(c->xyz, xyz_i);
      swap_buf(c->tets, tets_i);
      swap_buf(c->face_nodes, fn_i);
      swap_buf(c->face_opp, fo_i);
      c->reordered = true;
    }
    c->rep.reordered = c->reordered ? 1 : 0;
    FS_CUDA(cudaEventRecord(c->ev1, c->stream));
    FS_CUDA(cudaEventSynchronize(c->ev1));
    c->rep.t_faces_ms = elapsed(c->ev0, c->ev1);
    c->nf = nf;
    c->ni = ni;
    if (n_faces) *n_faces = nf;
    if (n_interior) *n_interior = ni;
    c->stage = kFaces;
    return FSFEM_OK;
  });
}

fsfem_status fsfem_get_faces(const fsfem_ctx* cc, int32_t* face_nodes, int32_t* face_tet, int32_t* face_opp) {
  fsfem_ctx* c = const_cast<fsfem_ctx*>(cc);
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kFaces) return fail(c, FSFEM_ERR_STATE, "build_faces first");
    const int32_t* fn = c->face_nodes.get();
    const int32_t* fo = c->face_opp.get();
    if (c->reordered) {  // back to the caller's node ids (the sorted triples are restored exactly)
      int32_t* t = c->tmp_i.ensure(5 * c->nf);
      perm_ids_device(c->iperm.get(), fn, t, 3 * c->nf, c->stream);
      perm_ids_device(c->iperm.get(), fo, t + 3 * c->nf, 2 * c->nf, c->stream);
      fn = t;
      fo = t + 3 * c->nf;
    }
    from_device(face_nodes, fn, sizeof(int32_t) * 3 * c->nf, c->stream);
    from_device(face_tet, c->face_tet.get(), sizeof(int32_t) * 2 * c->nf, c->stream);
    from_device(face_opp, fo, sizeof(int32_t) * 2 * c->nf, c->stream);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_assemble_csr(fsfem_ctx* c, double E, double nu, int64_t* row_begin, int64_t* n_rows, int64_t* nnz) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kFaces) return fail(c, FSFEM_ERR_STATE, "build_faces first");
    if (!(E > 0.0) || !(nu > -1.0 && nu < 0.5) || !std::isfinite(E))
      return fail(c, FSFEM_ERR_INVALID_ARG, "need E > 0 and -1 < nu < 0.5");
    if (!c->have_pattern) {
      FS_CUDA(cudaEventRecord(c->ev0, c->stream));
      c->h_flags[0] = kNoError;
      build_pattern_device(c->tets.get(), c->nt, c->tet_face.get(), c->tet_across.get(), c->n_lo, c->nloc, c->stream,
                           c->scratch, c->pat, c->h_flags, c->method == FSFEM_METHOD_FEM_T4);
      fsfem_status s = decode_flags(c, c->h_flags[0], "symbolic");
      if (s != FSFEM_OK) return s;
      const bool tet = c->method == FSFEM_METHOD_FEM_T4;
      build_assembly_tiles(c->pat, c->xyz.get(), tet ? c->tets.get() : c->face_nodes.get(),
                           tet ? nullptr : c->face_opp.get(), tet, c->scratch, c->h_flags, c->stream);
      s = decode_flags(c, c->h_flags[0], "assembly tiles");
      if (s != FSFEM_OK) return s;
      if (9 * c->pat.nblk >= (1LL << 31)) return fail(c, FSFEM_ERR_UNSUPPORTED, "nnz >= 2^31");
      FS_CUDA(cudaEventRecord(c->ev1, c->stream));
      FS_CUDA(cudaEventSynchronize(c->ev1));
      c->rep.t_symbolic_ms = elapsed(c->ev0, c->ev1);
      c->vals.ensure(9 * c->pat.nsb + 2);  // + slack for the SpMV bulk copies (pattern.cuh)
      c->have_pattern = true;
      c->halo_ready = false;
      if (c->nranks > 1) {
        // the exchange lists are agreed with the peers at the first pcg_solve (setup_halo)
        build_halo_device(c->pat, c->nn, c->ranges, c->halo_need, c->scratch, c->stream);
        build_overlap_chunks(c->pat, c->stream);
      }
      drop_graph(c);
    }
    const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double mu = E / (2.0 * (1.0 + nu));
    FS_CUDA(cudaEventRecord(c->ev0, c->stream));
    assemble_tiles_device(c->pat, c->xyz.get(), lam, mu, c->vals.get(), c->method == FSFEM_METHOD_FEM_T4, c->stream);
    FS_CUDA(cudaEventRecord(c->ev1, c->stream));
    FS_CUDA(cudaEventSynchronize(c->ev1));
    c->rep.t_numeric_ms = elapsed(c->ev0, c->ev1);
    c->E = E;
    c->nu = nu;
    c->rep.stored_blocks = c->pat.nsb;
    c->rep.transposed_blocks = c->pat.ntb;
    c->rep.spmv_kernel = spmv_kind(c->pat);
    // the gather kernel reads the transposed list (8 B per transposed block), the dataflow kernel
    // the slot of every stored block (4 B); its pushed products are intermediate traffic
    c->rep.spmv_bytes = 72 * c->pat.nsb + 4 * c->pat.nsb +
                        (c->rep.spmv_kernel == 2 ? 4 * c->pat.nsb : 8 * c->pat.ntb) + 16 * (c->nloc + 1) +
                        24 * c->nn + 24 * c->nloc;
    c->rep.assembly_bytes = 24 * c->nn + 16 * c->nt + 72 * c->pat.nsb;
    c->rep.assembly_aux_bytes = c->pat.tile_blob_bytes;
    if (row_begin) *row_begin = 3 * c->n_lo;
    if (n_rows) *n_rows = 3 * c->nloc;
    if (nnz) *nnz = 9 * c->pat.nblk;
    c->stage = kAssembled;
    return FSFEM_OK;
  });
}

fsfem_status fsfem_get_csr(const fsfem_ctx* cc, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  fsfem_ctx* c = const_cast<fsfem_ctx*>(cc);
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kAssembled) return fail(c, FSFEM_ERR_STATE, "assemble_csr first");
    const int64_t nnz = 9 * c->pat.nblk, nr = 3 * c->nloc;
    DevBuf<int64_t> rp;
    DevBuf<int32_t> ci;
    DevBuf<double> vo;
    int64_t* d_rp = nullptr;
    int32_t* d_ci = nullptr;
    double* d_vo = nullptr;
    if (row_ptr) d_rp = is_device_ptr(row_ptr) ? row_ptr : rp.ensure(nr + 1);
    if (col_idx) d_ci = is_device_ptr(col_idx) ? col_idx : ci.ensure(std::max<int64_t>(nnz, 1));
    if (vals) d_vo = is_device_ptr(vals) ? vals : vo.ensure(std::max<int64_t>(nnz, 1));
    if (c->nloc > 0 && c->reordered) {
      int64_t* t = c->exp_tmp.ensure(2 * (c->nn + 1));
      DevBuf<unsigned char> sc;
      const size_t tb = scan_tmp_bytes(c->nn + 1);
      sc.ensure(tb);
      export_csr_user_device(c->perm.get(), c->iperm.get(), c->pat, c->vals.get(), t, t + c->nn + 1, sc.get(), tb, d_rp,
                             d_ci, d_vo, c->stream);
      FS_CUDA(cudaStreamSynchronize(c->stream));
    } else if (c->nloc > 0) {
      export_csr_device(c->pat, c->vals.get(), d_rp, d_ci, d_vo, c->stream);
    }
    else if (d_rp) FS_CUDA(cudaMemsetAsync(d_rp, 0, sizeof(int64_t), c->stream));
    if (row_ptr && d_rp != row_ptr) from_device(row_ptr, d_rp, sizeof(int64_t) * (nr + 1), c->stream);
    if (col_idx && d_ci != col_idx) from_device(col_idx, d_ci, sizeof(int32_t) * nnz, c->stream);
    if (vals && d_vo != vals) from_device(vals, d_vo, sizeof(double) * nnz, c->stream);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_apply_bc(fsfem_ctx* c, const int32_t* dirichlet, int64_t n_dir, const double* loads, int mode,
                            double penalty_scale) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kAssembled) return fail(c, FSFEM_ERR_STATE, "assemble_csr first");
    if (c->stage >= kBc) return fail(c, FSFEM_ERR_STATE, "BCs already applied: re-assemble first");
    if (!loads || n_dir < 0 || (n_dir > 0 && !dirichlet) || (mode != 0 && mode != 1))
      return fail(c, FSFEM_ERR_INVALID_ARG, "bad dirichlet/loads/mode");
    if (mode == 1 && c->nranks > 1) return fail(c, FSFEM_ERR_UNSUPPORTED, "PENALTY mode is single-GPU only");
    const int64_t n = 3 * c->nloc;
    c->f.ensure(std::max<int64_t>(n, 1));
    c->dinv.ensure(std::max<int64_t>(n, 1));
    c->fixed.ensure(c->nn);
    c->staging.ensure(3 * c->nn);
    c->staging_i.ensure(std::max<int64_t>(n_dir, 1));
    FS_CUDA(cudaEventRecord(c->ev0, c->stream));
    node_in(c, loads, 3, c->staging.get());
    to_device(c->staging_i.get(), dirichlet, sizeof(int32_t) * n_dir, c->stream);
    if (c->reordered && n_dir > 0) {  // ids out of range are left for apply_bc to report
      int32_t* t = c->tmp_i.ensure(n_dir);
      FS_CUDA(cudaMemcpyAsync(t, c->staging_i.get(), sizeof(int32_t) * n_dir, cudaMemcpyDeviceToDevice, c->stream));
      perm_ids_valid_device(c->perm.get(), t, c->staging_i.get(), n_dir, c->nn, c->stream);
    }
    apply_bc_device(c->pat.sptr.get(), c->pat.snbr.get(), c->pat.sdiag.get(), c->n_lo, c->nloc, c->nn, c->staging_i.get(),
                    n_dir, c->staging.get(), mode, penalty_scale, c->vals.get(), c->f.get(), c->dinv.get(),
                    c->fixed.get(), c->flags.get(), c->stream);
    FS_CUDA(cudaEventRecord(c->ev1, c->stream));
    FS_CUDA(cudaMemcpyAsync(c->h_flags, c->flags.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    FS_CUDA(cudaStreamSynchronize(c->stream));
    fsfem_status s = decode_flags(c, c->h_flags[0], "apply_bc");
    if (s != FSFEM_OK) return s;
    c->rep.t_bc_ms = elapsed(c->ev0, c->ev1);
    c->stage = kBc;
    return FSFEM_OK;
  });
}

fsfem_status fsfem_spmv(fsfem_ctx* c, const double* p, double* q) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kAssembled) return fail(c, FSFEM_ERR_STATE, "assemble_csr first");
    if (!p || !q) return fail(c, FSFEM_ERR_INVALID_ARG, "null vector");
    c->x_full.ensure(3 * c->nn);
    c->q.ensure(std::max<int64_t>(3 * c->nloc, 1));
    node_in(c, p, 3, c->x_full.get());
    spmv_of(c, c->x_full.get(), c->q.get(), false);
    node_out(c, q, c->q.get(), c->n_lo, c->nloc, 3);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_pcg_solve(fsfem_ctx* c, double* u, int u0_is_zero, double rel_tol, int64_t max_iter,
                             fsfem_report* rep) {
  return guarded(c, [&]() -> fsfem_status {
    const Ranks cs = ranks_of(c);
    fsfem_ctx* c0 = cs[0];
    for (fsfem_ctx* r : cs) {
      if (r->stage < kBc) return fail(c, FSFEM_ERR_STATE, "apply_bc first (on every rank of the loopback group)");
      if (r->det != c0->det || r->exchange != c0->exchange || r->pcg_variant != c0->pcg_variant || r->nn != c0->nn)
        return fail(c, FSFEM_ERR_INVALID_ARG, "the ranks disagree on mode, exchange, variant or mesh");
    }
    if (c->nranks > 1 && !c->comm && !c->loop) return fail(c, FSFEM_ERR_STATE, "partition-only context: no communicator");
    if (!u) return fail(c, FSFEM_ERR_INVALID_ARG, "null u");
    const int64_t nglob = 3 * c->nn;
    if (rel_tol <= 0.0) rel_tol = 1e-10;
    if (max_iter <= 0) max_iter = std::max<int64_t>(1000, static_cast<int64_t>(20.0 * std::sqrt(double(nglob))));
    // recurrence: the standard form unless the single-reduction form is asked for (AUTO keeps the
    // standard one until the multi-GPU variants are measured); deterministic mode is standard
    const bool cg1 = !c0->det && c0->pcg_variant == FSFEM_PCG_SINGLE_REDUCTION;
    for (fsfem_ctx* r : cs) {
      const int64_t n = 3 * r->nloc;
      r->x_full.ensure(nglob);
      r->p_full.ensure(nglob);
      r->r.ensure(std::max<int64_t>(n, 1));
      r->q.ensure(std::max<int64_t>(n, 1));
      r->part.ensure(8 * static_cast<size_t>(pcg_grid()));  // SpMV / dot partials; [4g, 6g): update partials
      r->all.ensure(4 * static_cast<size_t>(r->nranks));
      if (r->det) r->dpart.ensure(3 * det_nchunks(r->nn));
      if (cg1) {
        r->cg_p.ensure(std::max<int64_t>(n, 1));
        r->cg_s.ensure(std::max<int64_t>(n, 1));
      }
      r->cg_active = cg1;
    }
    if (c0->nranks > 1 && c0->exchange == FSFEM_EXCHANGE_HALO && !c0->halo_ready) setup_halo(cs);
    const bool det = c0->det;
    const int64_t nchg = det ? det_nchunks(c0->nn) : 0;

    auto set_state = [&](int64_t budget) {
      for (fsfem_ctx* r : cs) {
        std::memset(r->h_st, 0, sizeof(PcgState));
        r->h_st->tol = rel_tol;
        r->h_st->max_iter = budget;
        r->h_st->nranks = det ? 1 : r->nranks;  // det: every rank sums all chunk partials itself
        r->h_st->variant = cg1 ? 1 : 0;
        r->h_st->cg_first = cg1 ? 1 : 0;
        r->h_st->upd_part = r->part.get() + 4 * pcg_grid();
        r->h_st->upd_n = cg_update_grid(3 * r->nloc);
        r->h_st->spmv_t0 = ~0ull;
        r->h_st->upd_t0 = ~0ull;
        FS_CUDA(cudaMemcpyAsync(r->st.get(), r->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, r->stream));
      }
    };
    // (Re)start from x_full (x0 = 0 or the current iterate): r = f - K x, z = D^-1 r, p = z.
    auto start = [&](bool x_is_zero) {
      for (fsfem_ctx* r : cs) {
        const double* q0 = nullptr;
        if (!x_is_zero) {
          spmv_of(r, r->x_full.get(), r->q.get(), false);
          q0 = r->q.get();
        }
        if (det)
          launch_det_dots(0, r->n_lo, r->nloc, r->f.get(), q0, r->dinv.get(), r->r.get(), own_p(r), nullptr,
                          r->st.get(), r->dpart.get(), r->stream);
        else
          launch_init(r->f.get(), q0, r->dinv.get(), r->r.get(), own_p(r), 3 * r->nloc, r->st.get(), r->part.get(),
                      r->stream);
      }
      if (det) {
        coll_dpart(cs);
        for (fsfem_ctx* r : cs) launch_det_finish(r->st.get(), r->dpart.get(), nchg, 0, r->stream);
      } else {
        coll_partials(cs, 0);
      }
      coll_full(cs, &fsfem_ctx::p_full);
      if (cg1) {  // p = s = 0, then w = K u and the first alpha (u = D^-1 r is in p_full)
        for (fsfem_ctx* r : cs) {
          FS_CUDA(cudaMemsetAsync(r->cg_p.get(), 0, sizeof(double) * std::max<int64_t>(3 * r->nloc, 1), r->stream));
          FS_CUDA(cudaMemsetAsync(r->cg_s.get(), 0, sizeof(double) * std::max<int64_t>(3 * r->nloc, 1), r->stream));
          spmv_of(r, r->p_full.get(), r->q.get(), true);
        }
        coll_partials(cs, 4);
      }
    };
    auto read_state = [&]() {
      FS_CUDA(cudaMemcpyAsync(c0->h_st, c0->st.get(), sizeof(PcgState), cudaMemcpyDeviceToHost, c0->stream));
      FS_CUDA(cudaStreamSynchronize(c0->stream));
    };

    FS_CUDA(cudaEventRecord(c->ev0, c->stream));
    set_state(max_iter);
    for (fsfem_ctx* r : cs) {
      FS_CUDA(cudaMemsetAsync(r->x_full.get(), 0, sizeof(double) * nglob, r->stream));
      FS_CUDA(cudaMemsetAsync(r->p_full.get(), 0, sizeof(double) * nglob, r->stream));
      if (!u0_is_zero) node_in(r, u, 3, r->x_full.get());
    }
    start(u0_is_zero != 0);
    read_state();

    // The loop: one cluster kernel (small meshes), a device-side while node, or host-polled
    // batches of kBatch iterations.
    const std::vector<uintptr_t> key = graph_key_of(cs);
    const bool cluster_ok = cs.size() == 1 && c->nranks == 1 && !det && !cg1;
    const bool cluster = cluster_ok && (c->loop_mode == FSFEM_LOOP_CLUSTER ||
                                        (c->loop_mode == FSFEM_LOOP_AUTO && c->pat.nsb + c->pat.ntb <= kClusterAutoBlocks));
    int cl_C = 0;
    if (cluster) {
      cl_C = cluster_pcg_size(c->nloc);
      c->cl_split.ensure(cl_C + 1);
      cluster_pcg_split(c->pat, cl_C, c->cl_split.get(), c->stream);
    }
    bool device_loop = !cluster && c->loop_mode == FSFEM_LOOP_DEVICE && !c->dgraph_failed && !(c0->nranks > 1 && !c0->loop);
    if (device_loop && (!c->dgraph || key != c->dgraph_key)) {
      if (c->dgraph) cudaGraphExecDestroy(c->dgraph);
      c->dgraph = nullptr;
      cudaGraph_t g;
      FS_CUDA(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle handle;
      FS_CUDA(cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = handle;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      FS_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      FS_CUDA(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      set_capturing(true);
      try {
        for (int it = 0; it < kDevBatch; ++it) pcg_iteration(cs, nullptr, nullptr);
        launch_loop_cond(handle, c0->st.get(), c->stream);
      } catch (...) {
        set_capturing(false);
        cudaGraph_t dummy;
        cudaStreamEndCapture(c->stream, &dummy);
        cudaGraphDestroy(g);
        throw;
      }
      set_capturing(false);
      cudaGraph_t captured;
      FS_CUDA(cudaStreamEndCapture(c->stream, &captured));
      c->dgraph_body_launches = captured_launches();
      if (cudaGraphInstantiate(&c->dgraph, g, 0) != cudaSuccess) {
        cudaGetLastError();
        c->dgraph = nullptr;
        c->dgraph_failed = true;  // fall back to host-polled batches from now on
        device_loop = false;
      } else {
        c->dgraph_key = key;
      }
      cudaGraphDestroy(g);
    }
    if (!cluster && !device_loop && (!c->graph || key != c->graph_key)) {
      if (c->graph) cudaGraphExecDestroy(c->graph);
      c->graph = nullptr;
      cudaGraph_t g;
      FS_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      set_capturing(true);
      try {
        // the second SpMV of every batch is bracketed by events (a live per-launch sample that
        // follows an update kernel, as every SpMV but the batch's first does; the first one also
        // carries the graph's launch latency); an event pair around every SpMV would cost ~14 us
        // per iteration at cfg4
        for (int it = 0; it < kBatch; ++it)
          pcg_iteration(cs, it == 1 ? c->spmv_ev[0] : nullptr, it == 1 ? c->spmv_ev[1] : nullptr);
      } catch (...) {
        set_capturing(false);
        cudaStreamEndCapture(c->stream, &g);
        throw;
      }
      set_capturing(false);
      FS_CUDA(cudaStreamEndCapture(c->stream, &g));
      FS_CUDA(cudaGraphInstantiate(&c->graph, g, 0));
      cudaGraphDestroy(g);
      c->graph_key = key;
      c->graph_launches = captured_launches();
    }
    int64_t total_iters = 0;
    int restarts = 0;
    double true_rel = 0.0, floor_rel = 0.0;
    double ev_ms = 0.0;
    int64_t ev_n = 0;
    for (;;) {
      if (cluster) {
        launch_pcg_cluster(c->pat, c->vals.get(), c->dinv.get(), own_x(c), c->r.get(), c->p_full.get(), c->q.get(),
                           c->cl_split.get(), cl_C, c->st.get(), c->stream);
        read_state();
      } else if (device_loop) {
        FS_CUDA(cudaGraphLaunch(c->dgraph, c->stream));
        read_state();
        const long long bodies = std::max<long long>(1, (c0->h_st->iters + kDevBatch - 1) / kDevBatch);
        count_launch(bodies * c->dgraph_body_launches);
      } else {
        while (c0->h_st->done_d == 0.0) {
          const long long before = c0->h_st->iters;
          FS_CUDA(cudaGraphLaunch(c->graph, c->stream));
          count_launch(c->graph_launches);
          read_state();
          if (c0->h_st->iters > before + 1) {  // the sampled SpMV (iteration 1 of the batch) ran
            ev_ms += elapsed(c->spmv_ev[0], c->spmv_ev[1]);
            ++ev_n;
          }
          if (c0->h_st->iters == before && c0->h_st->done_d == 0.0) throw Error(FSFEM_ERR_CUDA, "pcg made no progress");
        }
      }
      if (c0->h_st->done_d == 0.0) throw Error(FSFEM_ERR_CUDA, "pcg loop ended before the recurrence stopped");
      total_iters += c0->h_st->iters;
      // true residual ||f - K x|| / ||f|| and its rounding floor eps ||K||_F ||x|| / ||f||
      coll_allgatherv(cs, &fsfem_ctx::x_full);  // every rank holds the whole iterate
      for (fsfem_ctx* r : cs) {
        spmv_of(r, r->x_full.get(), r->q.get(), false);
        launch_sumsq(r->vals.get(), 9 * r->pat.nsb, r->st.get(), r->part.get(), r->stream);
      }
      if (det) {
        coll_partials(cs, 5);  // ||K||_F^2 bound: sum over ranks (no effect with one rank)
        for (fsfem_ctx* r : cs)
          launch_det_dots(3, r->n_lo, r->nloc, r->f.get(), r->q.get(), nullptr, nullptr, nullptr, own_x(r), r->st.get(),
                          r->dpart.get(), r->stream);
        coll_dpart(cs);
        for (fsfem_ctx* r : cs) launch_det_finish(r->st.get(), r->dpart.get(), nchg, 3, r->stream);
      } else {
        for (fsfem_ctx* r : cs) launch_resid(r->f.get(), r->q.get(), own_x(r), 3 * r->nloc, r->st.get(), r->part.get(), r->stream);
        coll_partials(cs, 3);
      }
      read_state();
      const PcgState& h = *c0->h_st;
      const double ff = h.ff;
      true_rel = ff > 0 ? std::sqrt(h.local[3] / ff) : 0.0;
      floor_rel = ff > 0 ? std::ldexp(1.0, -52) * std::sqrt(h.local[2]) * std::sqrt(h.local[1]) / std::sqrt(ff) : 0.0;
      const bool miss = h.status == FSFEM_OK && true_rel > std::max(rel_tol, floor_rel);
      if (!miss || restarts >= c->max_restarts || total_iters >= max_iter) {
        if (miss) {  // the recurrence converged but the true residual did not follow
          for (fsfem_ctx* r : cs) r->h_st->status = FSFEM_ERR_NOT_CONVERGED;
        }
        break;
      }
      // residual replacement: restart the recurrence from the current iterate (timers carry over)
      ++restarts;
      const unsigned long long tns = c0->h_st->spmv_ns, tcnt = c0->h_st->spmv_cnt;
      set_state(max_iter - total_iters);
      for (fsfem_ctx* r : cs) {
        r->h_st->spmv_ns = tns;
        r->h_st->spmv_cnt = tcnt;
        FS_CUDA(cudaMemcpyAsync(r->st.get(), r->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, r->stream));
      }
      for (fsfem_ctx* r : cs) FS_CUDA(cudaMemsetAsync(r->p_full.get(), 0, sizeof(double) * nglob, r->stream));
      start(false);
      read_state();
    }
    FS_CUDA(cudaEventRecord(c->ev1, c->stream));
    node_out(c0, u, c0->x_full.get(), 0, c->nn, 3);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    const PcgState& h = *c0->h_st;
    const int status = h.status;
    for (fsfem_ctx* r : cs) {
      r->rep.iterations = total_iters;
      r->rep.converged = (status == FSFEM_OK) ? 1 : 0;
      r->rep.rel_residual = h.ff > 0 ? std::sqrt(h.rr / h.ff) : 0.0;
      r->rep.true_rel_residual = true_rel;
      r->rep.residual_floor = floor_rel;
      r->rep.restarts = restarts;
      r->rep.t_pcg_ms = elapsed(c->ev0, c->ev1);
      r->rep.t_spmv_dev_ms = static_cast<double>(h.spmv_ns) * 1e-6;  // device timer, every PCG SpMV
      r->rep.spmv_dev_launches = static_cast<int64_t>(h.spmv_cnt);
      r->rep.t_spmv_ms = device_loop ? r->rep.t_spmv_dev_ms : ev_ms;  // CUDA events (host-polled loop)
      r->rep.spmv_launches = device_loop ? r->rep.spmv_dev_launches : ev_n;
      r->rep.pcg_loop = cluster ? FSFEM_LOOP_CLUSTER : (device_loop ? FSFEM_LOOP_DEVICE : FSFEM_LOOP_HOST);
      r->rep.kernel_launches = launch_count();
    }
    if (std::getenv("FSFEM_GAP_PRINT"))
      std::fprintf(stderr, "gap timing: spmv %.2f us, update %.2f us, spmv->update gap %.2f us (%llu updates)\n",
                   h.spmv_ns * 1e-3 / std::max(1ull, h.spmv_cnt), h.upd_ns * 1e-3 / std::max(1ull, h.upd_cnt),
                   h.gap_ns * 1e-3 / std::max(1ull, h.upd_cnt), h.upd_cnt);
    if (rep) *rep = c->rep;
    if (status == FSFEM_ERR_BREAKDOWN) return fail(c, FSFEM_ERR_BREAKDOWN, "pcg breakdown (p.q <= 0 or non-finite)");
    if (status == FSFEM_ERR_NOT_CONVERGED) {
      if (total_iters >= max_iter) return fail(c, FSFEM_ERR_NOT_CONVERGED, "pcg reached max_iter=" + std::to_string(max_iter));
      return fail(c, FSFEM_ERR_NOT_CONVERGED,
                  "true residual " + std::to_string(true_rel) + " above max(tol, rounding floor " +
                      std::to_string(floor_rel) + ") after " + std::to_string(restarts) + " restarts");
    }
    return FSFEM_OK;
  });
}

fsfem_status fsfem_recover_stress(fsfem_ctx* c, const double* u, double* strain, double* stress, double* node_stress,
                                  double* node_vm, int64_t* n_domains) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kAssembled) return fail(c, FSFEM_ERR_STATE, "assemble_csr first");
    if (!u) return fail(c, FSFEM_ERR_INVALID_ARG, "null u");
    const bool tet = c->method == FSFEM_METHOD_FEM_T4;
    const int64_t nd = tet ? c->nt : c->nf;
    if (n_domains) *n_domains = nd;
    const double lam = c->E * c->nu / ((1.0 + c->nu) * (1.0 - 2.0 * c->nu));
    const double mu = c->E / (2.0 * (1.0 + c->nu));
    c->rec_u.ensure(3 * c->nn);
    node_in(c, u, 3, c->rec_u.get());
    double* d_stress = (stress && is_device_ptr(stress)) ? stress : c->rec_stress.ensure(6 * nd);
    double* d_strain = nullptr;
    if (strain) d_strain = is_device_ptr(strain) ? strain : c->rec_strain.ensure(6 * nd);
    double* d_nodes = nullptr;
    if (node_stress) d_nodes = c->rec_nodes.ensure(std::max<int64_t>(6 * c->nloc, 1));
    double* d_vm = nullptr;
    if (node_vm) d_vm = c->rec_vm.ensure(std::max<int64_t>(c->nloc, 1));
    // per-domain records s_K, V (the assembly keeps them on chip; recovery recomputes them)
    c->face_s.ensure(16 * std::max(c->nf, c->nt));
    c->face_V.ensure(std::max(c->nf, c->nt));
    if (tet)
      tet_s_device(c->xyz.get(), c->tets.get(), c->nt, c->face_s.get(), c->face_V.get(), c->stream);
    else
      face_s_device(c->xyz.get(), c->tets.get(), c->face_nodes.get(), c->face_tet.get(), c->face_opp.get(), c->nf,
                    c->face_s.get(), c->face_V.get(), c->stream);
    recover_device(tet ? c->tets.get() : c->face_nodes.get(), tet ? nullptr : c->face_opp.get(), tet, c->face_s.get(),
                   c->face_V.get(), nd,
                   c->pat.nf_ptr.get(), c->pat.nf_idx.get(), c->nloc, c->rec_u.get(), lam, mu, d_strain, d_stress,
                   d_nodes, d_vm, c->stream);
    if (stress && d_stress != stress) from_device(stress, d_stress, sizeof(double) * 6 * nd, c->stream);
    if (strain && d_strain != strain) from_device(strain, d_strain, sizeof(double) * 6 * nd, c->stream);
    if (node_stress) node_out(c, node_stress, d_nodes, c->n_lo, c->nloc, 6);
    if (node_vm) node_out(c, node_vm, d_vm, c->n_lo, c->nloc, 1);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_domain_stiffness(fsfem_ctx* c, const int64_t* ids, int64_t n, double* K, int32_t* field) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kAssembled) return fail(c, FSFEM_ERR_STATE, "assemble_csr first (uses its E, nu)");
    if (n < 0 || (n > 0 && (!ids || !K))) return fail(c, FSFEM_ERR_INVALID_ARG, "null ids / K or n < 0");
    if (n == 0) return FSFEM_OK;
    const bool tet = c->method == FSFEM_METHOD_FEM_T4;
    const int64_t nd = tet ? c->nt : c->nf;
    for (int64_t q = 0; q < n; ++q)  // argument check
      if (ids[q] < 0 || ids[q] >= nd) return fail(c, FSFEM_ERR_INVALID_ARG, "domain id out of range");
    const double lam = c->E * c->nu / ((1.0 + c->nu) * (1.0 - 2.0 * c->nu));
    const double mu = c->E / (2.0 * (1.0 + c->nu));
    DevBuf<int64_t> d_ids;
    DevBuf<double> d_K;
    DevBuf<int32_t> d_f, d_f2;
    d_ids.ensure(n);
    d_K.ensure(225 * n);
    d_f.ensure(5 * n);
    to_device(d_ids.get(), ids, sizeof(int64_t) * n, c->stream);
    domain_stiffness_device(c->xyz.get(), tet ? c->tets.get() : c->face_nodes.get(), tet ? nullptr : c->face_opp.get(),
                            tet, d_ids.get(), n, lam, mu, d_K.get(), d_f.get(), c->stream);
    const int32_t* fo = d_f.get();
    if (c->reordered) {  // back to the caller's node ids
      d_f2.ensure(5 * n);
      perm_ids_device(c->iperm.get(), fo, d_f2.get(), 5 * n, c->stream);
      fo = d_f2.get();
    }
    from_device(K, d_K.get(), sizeof(double) * 225 * n, c->stream);
    if (field) from_device(field, fo, sizeof(int32_t) * 5 * n, c->stream);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_surface_loads(fsfem_ctx* c, const uint8_t* node_flag, const double* traction, double* loads) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kAssembled) return fail(c, FSFEM_ERR_STATE, "assemble_csr first (uses its node lists)");
    if (!node_flag || !traction || !loads) return fail(c, FSFEM_ERR_INVALID_ARG, "null argument");
    c->fixed.ensure(c->nn);
    if (c->reordered) {
      uint8_t* t = c->tmp_u8.ensure(c->nn);
      to_device(t, node_flag, c->nn, c->stream);
      permute_rows_u8_device(c->iperm.get(), t, c->fixed.get(), c->nn, true, c->stream);
    } else {
      to_device(c->fixed.get(), node_flag, c->nn, c->stream);
    }
    double* d_loads = c->rec_u.ensure(std::max<int64_t>(3 * c->nn, 1));
    surface_loads_device(c->pat.nf_ptr.get(), c->pat.nf_idx.get(), c->method == FSFEM_METHOD_FEM_T4, c->tet_face.get(),
                         c->face_nodes.get(), c->face_tet.get(), c->fixed.get(), c->xyz.get(), c->n_lo, c->nloc,
                         traction, d_loads, c->stream);
    node_out(c, loads, d_loads, c->n_lo, c->nloc, 3);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_get_report(const fsfem_ctx* c, fsfem_report* rep) {
  if (!c || !rep) return FSFEM_ERR_INVALID_ARG;
  *rep = c->rep;
  return FSFEM_OK;
}

}  // extern "C"
