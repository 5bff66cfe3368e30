// C ABI of the FS-FEM hot path (include/fsfem.h): context, call-order state machine,
// host/device pointer handling, stage timing, PCG batching in CUDA graphs, NCCL row partition.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstring>
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
                        DevBuf<int32_t>& face_opp, DevBuf<int32_t>& tet_face, int64_t* n_faces, int64_t* n_interior,
                        unsigned long long* h_flags);
void build_pattern_device(const int32_t* d_tets, int64_t nt, const int32_t* tet_face, const int32_t* face_tet,
                          const int32_t* face_opp, int64_t n_lo, int64_t nloc, cudaStream_t s,
                          DevBuf<unsigned char>& scratch, Pattern& pat, unsigned long long* h_flags, int fem);
void export_csr_device(const Pattern& pat, const double* svals, int64_t* row_ptr, int32_t* col_idx, double* vals,
                       cudaStream_t s);
void face_s_device(const double* xyz, const int32_t* tets, const int32_t* face_nodes, const int32_t* face_tet,
                   const int32_t* face_opp, int64_t nf, double* face_s, double* face_V, cudaStream_t s);
void build_halo_device(Pattern& pat, int64_t nn, int64_t chunk, int nranks, std::vector<int64_t>& need,
                       DevBuf<unsigned char>& scratch, cudaStream_t s);
void halo_pack_device(const double* full, const int32_t* nodes, int64_t n, double* buf, cudaStream_t s);
void halo_unpack_device(const double* buf, const int32_t* nodes, int64_t n, double* full, cudaStream_t s);
void build_assembly_program(Pattern& pat, const int32_t* rec_a, const int32_t* rec_b, bool tet,
                            DevBuf<unsigned char>& scratch, unsigned long long* h_flags, cudaStream_t s);
void assemble_rows_device(const Pattern& pat, const int32_t* face_nodes, const int32_t* face_opp,
                          const double* face_s, double lam, double mu, double* vals, bool tet, cudaStream_t s);
void tet_s_device(const double* xyz, const int32_t* tets, int64_t nt, double* tet_s, double* tet_V, cudaStream_t s);
void recover_device(const int32_t* rec_a, const int32_t* rec_b, bool tet, const double* rec_s, const double* rec_V,
                    int64_t nrec,
                    const int64_t* nd_ptr, const int32_t* nd_idx, int64_t nloc, const double* u, double lam, double mu,
                    double* strain, double* stress, double* node_stress, double* node_vm, cudaStream_t s);
double mean_tet_span_device(const int32_t* tets, int64_t nt, unsigned long long* d_tmp, cudaStream_t s);
void morton_order_device(const double* d_xyz, int64_t nn, int32_t* iperm, int32_t* perm, DevBuf<unsigned char>& scratch,
                         cudaStream_t s);
void perm_ids_device(const int32_t* perm, const int32_t* in, int32_t* out, int64_t n, cudaStream_t s);
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
void count_launch(long long n) {
  if (!g_capturing) g_launches.fetch_add(n, std::memory_order_relaxed);
}
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
void set_capturing(bool on) { g_capturing = on; }

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

// ---- NCCL, resolved at run time (torch has already loaded libnccl.so.2 in practice) ----
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
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
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GetErrorString;
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.p2p = api.Send && api.Recv && api.GroupStart && api.GroupEnd;
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

struct fsfem_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int stage = kCreated;
  // partition
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  int64_t n_lo = 0, nloc = 0, chunk = 0;
  // mesh
  int64_t nn = 0, nt = 0, nf = 0, ni = 0;
  DevBuf<double> xyz;
  DevBuf<int32_t> tets;
  DevBuf<int32_t> face_nodes, face_tet, face_opp, tet_face;
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
  // graph cache
  cudaGraphExec_t graph = nullptr;
  int graph_batch = 0;
  const void* graph_key[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

constexpr int kBatch = 32;  // PCG iterations per CUDA graph launch

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
}

// allgather of the 4 per-rank partials and the combine step (multi-rank only)
void combine(fsfem_ctx* c, int stage) {
  FS_NCCL(nccl().AllGather(c->st.get()->local, c->all.get(), 4, ncclDouble, c->comm, c->stream));
  launch_combine(c->st.get(), c->all.get(), stage, c->stream);
}

// p_full own slice -> everyone (in-place allgather, equal padded slices)
void allgather_full(fsfem_ctx* c, double* full) {
  if (c->nranks == 1) return;
  FS_NCCL(nccl().AllGather(full + 3 * c->chunk * c->rank, full, 3 * c->chunk, ncclDouble, c->comm, c->stream));
}

// Halo mode: each rank receives only the entries of its halo (halo.cu) from their owners and
// sends the entries its peers need; the other remote entries of `full` are left stale (the SpMV
// never reads them).  Fixed send/recv sizes per peer, agreed once per pattern (setup_halo).
void halo_exchange(fsfem_ctx* c, double* full) {
  const int nr = c->nranks;
  int64_t ns = 0;
  for (int q = 0; q < nr; ++q) ns += c->halo_send[q];
  halo_pack_device(full, c->halo_send_nodes.get(), ns, c->halo_sbuf.get(), c->stream);
  FS_NCCL(nccl().GroupStart());
  int64_t so = 0, ro = 0;
  for (int q = 0; q < nr; ++q) {
    if (c->halo_send[q] > 0)
      FS_NCCL(nccl().Send(c->halo_sbuf.get() + 3 * so, 3 * c->halo_send[q], ncclDouble, q, c->comm, c->stream));
    if (c->halo_need[q] > 0)
      FS_NCCL(nccl().Recv(c->halo_rbuf.get() + 3 * ro, 3 * c->halo_need[q], ncclDouble, q, c->comm, c->stream));
    so += c->halo_send[q];
    ro += c->halo_need[q];
  }
  FS_NCCL(nccl().GroupEnd());
  halo_unpack_device(c->halo_rbuf.get(), c->pat.halo.get(), c->pat.nhalo, full, c->stream);
}

// The search direction (p, or u in the single-reduction form) before an SpMV.
void gather_full(fsfem_ctx* c, double* full) {
  if (c->nranks == 1) return;
  if (c->exchange == FSFEM_EXCHANGE_HALO && c->halo_ready) halo_exchange(c, full);
  else allgather_full(c, full);
}

// Agree on the halo exchange with the peers (once per pattern): all-gather of the per-peer
// counts, then every rank sends each owner the list of that owner's nodes it needs.
void setup_halo(fsfem_ctx* c) {
  const int nr = c->nranks, me = c->rank;
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

// Single-reduction iteration (Chronopoulos-Gear): update (x, r, u = D^-1 r,
// p, s; partials of r.u and r.r), [all-gather of u], SpMV w = K u with u.w, and ONE combined
// reduction (u.w, r.u, r.r) -> alpha, beta.  p_full holds u, q holds w.
void pcg_iteration_cg(fsfem_ctx* c, cudaEvent_t e0, cudaEvent_t e1) {
  PcgState* st = c->st.get();
  double* own_u = c->p_full.get() + 3 * c->n_lo;
  double* own_x = c->x_full.get() + 3 * c->n_lo;
  const int64_t n = 3 * c->nloc;
  launch_cg_update(own_x, c->r.get(), own_u, c->cg_p.get(), c->cg_s.get(), c->q.get(), c->dinv.get(), n, st,
                   c->part.get() + 4 * pcg_grid(), c->stream);
  if (c->nranks > 1) gather_full(c, c->p_full.get());
  if (e0) FS_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
  launch_spmv(c->pat, c->vals.get(), c->p_full.get(), 3 * c->n_lo, c->q.get(), st, c->part.get(), true, c->stream);
  if (e1) FS_CUDA(cudaEventRecordWithFlags(e1, c->stream, cudaEventRecordExternal));
  if (c->nranks > 1) combine(c, 4);
}

void pcg_iteration(fsfem_ctx* c, cudaEvent_t e0, cudaEvent_t e1) {
  if (c->cg_active) {
    pcg_iteration_cg(c, e0, e1);
    return;
  }
  PcgState* st = c->st.get();
  double* own_p = c->p_full.get() + 3 * c->n_lo;
  double* own_x = c->x_full.get() + 3 * c->n_lo;
  const int64_t n = 3 * c->nloc;
  if (e0) FS_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
  launch_spmv(c->pat, c->vals.get(), c->p_full.get(), 3 * c->n_lo, c->q.get(), st, c->part.get(), true, c->stream);
  if (e1) FS_CUDA(cudaEventRecordWithFlags(e1, c->stream, cudaEventRecordExternal));
  if (c->nranks > 1) combine(c, 1);
  if (c->nranks == 1) {
    launch_update_direction(own_x, c->r.get(), own_p, c->q.get(), c->dinv.get(), n, st, c->part.get(), c->stream);
    return;
  }
  launch_update(own_x, c->r.get(), own_p, c->q.get(), c->dinv.get(), n, st, c->part.get(), c->stream);
  combine(c, 2);
  launch_direction(own_p, c->r.get(), c->dinv.get(), n, st, c->stream);
  gather_full(c, c->p_full.get());
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
    c->nn = n_nodes;
    c->nt = n_tets;
    c->chunk = ceil_div(n_nodes, c->nranks);
    c->n_lo = std::min<int64_t>(n_nodes, c->chunk * c->rank);
    c->nloc = std::min<int64_t>(n_nodes, c->n_lo + c->chunk) - c->n_lo;
    c->xyz.ensure(3 * n_nodes);
    c->tets.ensure(4 * n_tets);
    FS_CUDA(cudaEventRecord(c->ev0, c->stream));
    to_device(c->xyz.get(), xyz, sizeof(double) * 3 * n_nodes, c->stream);
    to_device(c->tets.get(), tets, sizeof(int32_t) * 4 * n_tets, c->stream);
    int64_t nf = 0, ni = 0;
    c->h_flags[0] = kNoError;
    build_faces_device(c->xyz.get(), n_nodes, c->tets.get(), n_tets, c->stream, c->scratch, c->face_nodes, c->face_tet,
                       c->face_opp, c->tet_face, &nf, &ni, c->h_flags);
    fsfem_status s = decode_flags(c, c->h_flags[0], "build_faces");
    if (s != FSFEM_OK) return s;
    // Internal node order (reorder.cu): renumber in Morton order when the caller's numbering is
    // not banded (mean tet id span > 16 N^(2/3)), never with several ranks (the documented row
    // partition is in the caller's numbering).
    c->span_tmp.ensure(1);
    c->mean_span = mean_tet_span_device(c->tets.get(), n_tets, c->span_tmp.get(), c->stream);
    const bool want = c->nranks == 1 &&
                      (c->reorder_mode == 1 ||
                       (c->reorder_mode == 0 && c->mean_span > 16.0 * std::pow(static_cast<double>(n_nodes), 2.0 / 3.0)));
    c->reordered = false;
    if (want) {
      c->iperm.ensure(n_nodes);
      c->perm.ensure(n_nodes);
      morton_order_device(c->xyz.get(), n_nodes, c->iperm.get(), c->perm.get(), c->scratch, c->stream);
      // the matrix path works on the renumbered mesh; faces keep their ids and order
      DevBuf<double> xyz_i;
      xyz_i.ensure(3 * n_nodes);
      permute_rows_device(c->iperm.get(), c->xyz.get(), xyz_i.get(), n_nodes, 3, true, c->stream);
      DevBuf<int32_t> tets_i, fn_i, fo_i;
      tets_i.ensure(4 * n_tets);
      fn_i.ensure(3 * nf);
      fo_i.ensure(2 * nf);
      perm_ids_device(c->perm.get(), c->tets.get(), tets_i.get(), 4 * n_tets, c->stream);
      perm_ids_device(c->perm.get(), c->face_nodes.get(), fn_i.get(), 3 * nf, c->stream);
      perm_ids_device(c->perm.get(), c->face_opp.get(), fo_i.get(), 2 * nf, c->stream);
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
      build_pattern_device(c->tets.get(), c->nt, c->tet_face.get(), c->face_tet.get(), c->face_opp.get(), c->n_lo,
                           c->nloc, c->stream, c->scratch, c->pat, c->h_flags, c->method == FSFEM_METHOD_FEM_T4);
      fsfem_status s = decode_flags(c, c->h_flags[0], "symbolic");
      if (s != FSFEM_OK) return s;
      const bool tet = c->method == FSFEM_METHOD_FEM_T4;
      build_assembly_program(c->pat, tet ? c->tets.get() : c->face_nodes.get(), tet ? nullptr : c->face_opp.get(), tet,
                             c->scratch, c->h_flags, c->stream);
      s = decode_flags(c, c->h_flags[0], "assembly program");
      if (s != FSFEM_OK) return s;
      if (9 * c->pat.nblk >= (1LL << 31)) return fail(c, FSFEM_ERR_UNSUPPORTED, "nnz >= 2^31");
      FS_CUDA(cudaEventRecord(c->ev1, c->stream));
      FS_CUDA(cudaEventSynchronize(c->ev1));
      c->rep.t_symbolic_ms = elapsed(c->ev0, c->ev1);
      c->vals.ensure(9 * c->pat.nsb + 2);  // + slack for the SpMV bulk copies (pattern.cuh)
      c->face_s.ensure(16 * std::max(c->nf, c->nt));
      c->face_V.ensure(std::max(c->nf, c->nt));
      c->have_pattern = true;
      c->halo_ready = false;
      if (c->nranks > 1) {
        build_halo_device(c->pat, c->nn, c->chunk, c->nranks, c->halo_need, c->scratch, c->stream);
        if (c->comm && c->exchange == FSFEM_EXCHANGE_HALO) {
          if (!nccl().p2p) return fail(c, FSFEM_ERR_NCCL, "ncclSend/ncclRecv not available for the halo exchange");
          setup_halo(c);
        }
      }
      drop_graph(c);
    }
    const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double mu = E / (2.0 * (1.0 + nu));
    FS_CUDA(cudaEventRecord(c->ev0, c->stream));
    if (c->method == FSFEM_METHOD_FEM_T4) {
      tet_s_device(c->xyz.get(), c->tets.get(), c->nt, c->face_s.get(), c->face_V.get(), c->stream);
      assemble_rows_device(c->pat, c->tets.get(), nullptr, c->face_s.get(), lam, mu, c->vals.get(), true, c->stream);
    } else {
      face_s_device(c->xyz.get(), c->tets.get(), c->face_nodes.get(), c->face_tet.get(), c->face_opp.get(), c->nf,
                    c->face_s.get(), c->face_V.get(), c->stream);
      assemble_rows_device(c->pat, c->face_nodes.get(), c->face_opp.get(), c->face_s.get(), lam, mu, c->vals.get(),
                           false, c->stream);
    }
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
    const int64_t nfull = 3 * c->chunk * c->nranks;
    c->x_full.ensure(nfull);
    c->q.ensure(std::max<int64_t>(3 * c->nloc, 1));
    node_in(c, p, 3, c->x_full.get());
    launch_spmv(c->pat, c->vals.get(), c->x_full.get(), 3 * c->n_lo, c->q.get(), nullptr, nullptr, false, c->stream);
    node_out(c, q, c->q.get(), c->n_lo, c->nloc, 3);
    FS_CUDA(cudaStreamSynchronize(c->stream));
    return FSFEM_OK;
  });
}

fsfem_status fsfem_pcg_solve(fsfem_ctx* c, double* u, int u0_is_zero, double rel_tol, int64_t max_iter,
                             fsfem_report* rep) {
  return guarded(c, [&]() -> fsfem_status {
    if (c->stage < kBc) return fail(c, FSFEM_ERR_STATE, "apply_bc first");
    if (c->nranks > 1 && !c->comm) return fail(c, FSFEM_ERR_STATE, "partition-only context: no communicator");
    if (!u) return fail(c, FSFEM_ERR_INVALID_ARG, "null u");
    const int64_t n = 3 * c->nloc;
    const int64_t nglob = 3 * c->nn;
    const int64_t nfull = 3 * c->chunk * c->nranks;
    if (rel_tol <= 0.0) rel_tol = 1e-10;
    if (max_iter <= 0) max_iter = std::max<int64_t>(1000, static_cast<int64_t>(20.0 * std::sqrt(double(nglob))));
    c->x_full.ensure(nfull);
    c->p_full.ensure(nfull);
    c->r.ensure(std::max<int64_t>(n, 1));
    c->q.ensure(std::max<int64_t>(n, 1));
    c->part.ensure(8 * static_cast<size_t>(pcg_grid()));  // SpMV / dot partials; [4g, 6g): update partials
    c->all.ensure(4 * static_cast<size_t>(c->nranks));
    PcgState* st = c->st.get();
    std::memset(c->h_st, 0, sizeof(PcgState));
    c->h_st->tol = rel_tol;
    c->h_st->max_iter = max_iter;
    c->h_st->nranks = c->nranks;
    // auto: one collective per iteration on several GPUs, the standard recurrence on one
    const bool cg1 = c->pcg_variant == FSFEM_PCG_SINGLE_REDUCTION ||
                     (c->pcg_variant == FSFEM_PCG_AUTO && c->nranks > 1);
    if (cg1 != c->cg_active) drop_graph(c);
    c->cg_active = cg1;
    c->h_st->variant = cg1 ? 1 : 0;
    c->h_st->cg_first = cg1 ? 1 : 0;
    c->h_st->upd_part = c->part.get() + 4 * pcg_grid();
    c->h_st->upd_n = cg_update_grid(n);
    if (cg1) {
      c->cg_p.ensure(std::max<int64_t>(n, 1));
      c->cg_s.ensure(std::max<int64_t>(n, 1));
    }

    FS_CUDA(cudaEventRecord(c->ev0, c->stream));
    FS_CUDA(cudaMemcpyAsync(st, c->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, c->stream));
    FS_CUDA(cudaMemsetAsync(c->x_full.get(), 0, sizeof(double) * nfull, c->stream));
    FS_CUDA(cudaMemsetAsync(c->p_full.get(), 0, sizeof(double) * nfull, c->stream));
    double* own_x = c->x_full.get() + 3 * c->n_lo;
    double* own_p = c->p_full.get() + 3 * c->n_lo;
    const double* q0 = nullptr;
    if (!u0_is_zero) {
      node_in(c, u, 3, c->x_full.get());
      launch_spmv(c->pat, c->vals.get(), c->x_full.get(), 3 * c->n_lo, c->q.get(), nullptr, nullptr, false, c->stream);
      q0 = c->q.get();
    }
    launch_init(c->f.get(), q0, c->dinv.get(), c->r.get(), own_p, n, st, c->part.get(), c->stream);
    if (c->nranks > 1) {
      combine(c, 0);
      gather_full(c, c->p_full.get());
    }
    if (cg1) {  // p = s = 0, then w = K u and the first alpha (u = D^-1 r is in p_full)
      FS_CUDA(cudaMemsetAsync(c->cg_p.get(), 0, sizeof(double) * std::max<int64_t>(n, 1), c->stream));
      FS_CUDA(cudaMemsetAsync(c->cg_s.get(), 0, sizeof(double) * std::max<int64_t>(n, 1), c->stream));
      launch_spmv(c->pat, c->vals.get(), c->p_full.get(), 3 * c->n_lo, c->q.get(), st, c->part.get(), true, c->stream);
      if (c->nranks > 1) combine(c, 4);
    }
    FS_CUDA(cudaMemcpyAsync(c->h_st, st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    FS_CUDA(cudaStreamSynchronize(c->stream));

    // graph of kBatch iterations with event pairs around each SpMV
    const void* key[4] = {c->vals.get(), c->x_full.get(), c->p_full.get(), c->r.get()};
    if (!c->graph || std::memcmp(key, c->graph_key, sizeof(key)) != 0) {
      drop_graph(c);
      cudaGraph_t g;
      FS_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      set_capturing(true);
      try {
        // One SpMV per batch is bracketed by events (a live per-launch sample for the roofline);
        // an event pair around every SpMV would cost ~14 us per iteration at cfg4.
        for (int it = 0; it < kBatch; ++it)
          pcg_iteration(c, it == 0 ? c->spmv_ev[0] : nullptr, it == 0 ? c->spmv_ev[1] : nullptr);
      } catch (...) {
        set_capturing(false);
        cudaStreamEndCapture(c->stream, &g);
        throw;
      }
      set_capturing(false);
      FS_CUDA(cudaStreamEndCapture(c->stream, &g));
      FS_CUDA(cudaGraphInstantiate(&c->graph, g, 0));
      cudaGraphDestroy(g);
      std::memcpy(c->graph_key, key, sizeof(key));
    }
    double spmv_ms = 0.0;
    int64_t spmv_n = 0;
    while (c->h_st->done_d == 0.0) {
      const long long before = c->h_st->iters;
      FS_CUDA(cudaGraphLaunch(c->graph, c->stream));
      count_launch((c->nranks > 1 ? (cg1 ? 3 : 5) : 2) * kBatch);
      FS_CUDA(cudaMemcpyAsync(c->h_st, st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
      FS_CUDA(cudaStreamSynchronize(c->stream));
      const long long ran = std::min<long long>(kBatch, c->h_st->iters - before);
      if (ran > 0) {  // the sampled SpMV ran (iteration 0 of the batch)
        spmv_ms += elapsed(c->spmv_ev[0], c->spmv_ev[1]);
        ++spmv_n;
      }
      if (c->h_st->iters == before && c->h_st->done_d == 0.0) throw Error(FSFEM_ERR_CUDA, "pcg made no progress");
    }
    FS_CUDA(cudaEventRecord(c->ev1, c->stream));
    // true residual ||f - K x|| / ||f||
    allgather_full(c, c->x_full.get());  // every rank returns the whole solution
    launch_spmv(c->pat, c->vals.get(), c->x_full.get(), 3 * c->n_lo, c->q.get(), nullptr, nullptr, false, c->stream);
    launch_resid(c->f.get(), c->q.get(), n, st, c->part.get(), c->stream);
    if (c->nranks > 1) combine(c, 3);
    node_out(c, u, c->x_full.get(), 0, c->nn, 3);
    FS_CUDA(cudaMemcpyAsync(c->h_st, st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    FS_CUDA(cudaStreamSynchronize(c->stream));
    (void)own_x;
    const PcgState& h = *c->h_st;
    c->rep.iterations = h.iters;
    c->rep.converged = (h.status == FSFEM_OK) ? 1 : 0;
    c->rep.rel_residual = h.ff > 0 ? std::sqrt(h.rr / h.ff) : 0.0;
    c->rep.true_rel_residual = h.ff > 0 ? std::sqrt(h.local[3] / h.ff) : 0.0;
    c->rep.t_pcg_ms = elapsed(c->ev0, c->ev1);
    c->rep.t_spmv_ms = spmv_ms;
    c->rep.spmv_launches = spmv_n;
    c->rep.kernel_launches = launch_count();
    if (rep) *rep = c->rep;
    if (h.status == FSFEM_ERR_BREAKDOWN) return fail(c, FSFEM_ERR_BREAKDOWN, "pcg breakdown (p.q <= 0 or non-finite)");
    if (h.status == FSFEM_ERR_NOT_CONVERGED)
      return fail(c, FSFEM_ERR_NOT_CONVERGED, "pcg reached max_iter=" + std::to_string(max_iter));
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
