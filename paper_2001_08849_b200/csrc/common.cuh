// Shared device/host helpers of the sm_100a FS-FEM path (no method arithmetic here).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "fsfem.h"

namespace fsfem {

constexpr int kWarp = 32;

// Host-side error carrying an fsfem_status; caught at the C ABI boundary.
struct Error : std::runtime_error {
  fsfem_status code;
  Error(fsfem_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FS_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      throw ::fsfem::Error(e_ == cudaErrorMemoryAllocation ? FSFEM_ERR_OOM : FSFEM_ERR_CUDA,   \
                           std::string(#call) + ": " + cudaGetErrorString(e_));                \
    }                                                                                          \
  } while (0)

// Process-wide count of kernels launched by the library (graph replays add their kernels).
void count_launch(long long n = 1);
long long launch_count();
void set_capturing(bool on);
long long captured_launches();

#define FS_LAUNCH_CHECK()              \
  do {                                 \
    FS_CUDA(cudaGetLastError());       \
    ::fsfem::count_launch();           \
  } while (0)

// Grow-only device buffer owned by the context.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* ensure(size_t count) {
    if (count > n) {
      release();
      size_t bytes = count * sizeof(T);
      if (bytes == 0) bytes = sizeof(T);
      FS_CUDA(cudaMalloc(&p, bytes));
      n = count;
    }
    return p;
  }
  T* get() const { return p; }
};

// Device error word: the first error (lowest code, then lowest index) wins, atomically.
// Layout: high 8 bits = fsfem_status, low 56 bits = index of the offending item.
__device__ __forceinline__ void report_error(unsigned long long* err, int code, long long idx) {
  unsigned long long v = (static_cast<unsigned long long>(code) << 56) | (static_cast<unsigned long long>(idx) & ((1ull << 56) - 1));
  atomicMin(err, v);
}
constexpr unsigned long long kNoError = ~0ull;

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Launch-shape helper: number of SMs of the current device (cached by the context).
int num_sms();

// Host phase timer for the cold path (FSFEM_PHASE_TIMES=1: every mark synchronises the stream
// and prints the wall time since the previous mark to stderr; otherwise a no-op).
struct PhaseTimer {
  cudaStream_t s;
  const char* tag;
  bool on;
  long long t0;
  PhaseTimer(cudaStream_t st, const char* tg);
  void mark(const char* name);
};

// ---- scan / reduce primitives (scan.cu) ----
// Exclusive prefix sum of in[0..n) into out[0..n], out[n] = total.  Deterministic.
void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s, void* tmp, size_t tmp_bytes);
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s, void* tmp, size_t tmp_bytes);
void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s, void* tmp,
                               size_t tmp_bytes);
size_t scan_tmp_bytes(int64_t n);

}  // namespace fsfem
