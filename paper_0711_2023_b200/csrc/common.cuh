// common.cuh -- shared host/device utilities of libtucker (no method arithmetic).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tucker.h"

namespace tk {

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error{code, msg}; }

#define TK_CUDA(x)                                                                           \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) {                                                                 \
      ::tk::fail(e_ == cudaErrorMemoryAllocation ? TUCKER_E_OOM : TUCKER_E_CUDA,             \
                 std::string(#x) + ": " + cudaGetErrorString(e_) + " at " + __FILE__ + ":" + \
                     std::to_string(__LINE__));                                              \
    }                                                                                        \
  } while (0)

// Launch counter shared by all launches of one handle (reported by tucker_stats).
extern thread_local int64_t* g_launch_counter;
// Stream of the handle call in progress: DBuf allocations are stream-ordered on
// it (cudaMallocAsync from the device's default pool, which keeps freed memory
// for reuse), so per-call temporaries cost no synchronous cudaMalloc/cudaFree.
// nullptr (no handle call, e.g. unit-test entry points): plain cudaMalloc.
extern thread_local cudaStream_t g_alloc_stream;
void mempool_retain(int device);  // default pool keeps freed memory (once per device)
// SMs held by a concurrent kernel of the calling handle (MP overlap): persistent grids size to
// (SMs - g_sm_reserve) so no block waits for a held SM's slots
extern thread_local int g_sm_reserve;
// when set, the one-CTA direct eigensolver records this event right after its kernel (the MP overlap's
// accounting: the solver kernel's own time, apart from the small kernels queued behind it)
extern thread_local cudaEvent_t g_eig_kernel_event;

bool sync_check_enabled();  // env TUCKER_SYNC_CHECK: synchronise + check after every launch

// Dynamic shared-memory opt-in (cudaFuncAttributeMaxDynamicSharedMemorySize) is
// a per-device setting: raise it for `fn` on the CURRENT device whenever `bytes`
// exceeds what was set there before (cached per (kernel, device), thread safe).
void smem_optin(const void* fn, size_t bytes);

#define TK_LAUNCH(kernel, grid, block, smem, stream, ...)                 \
  do {                                                                    \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);           \
    TK_CUDA(cudaGetLastError());                                          \
    if (::tk::g_launch_counter) ++(*::tk::g_launch_counter);              \
    if (::tk::sync_check_enabled()) {                                     \
      cudaError_t se_ = cudaStreamSynchronize(stream);                    \
      if (se_ != cudaSuccess)                                             \
        ::tk::fail(TUCKER_E_CUDA, std::string("kernel ") + #kernel +      \
                   " failed: " + cudaGetErrorString(se_));                \
    }                                                                     \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// RAII device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;  // stream of a stream-ordered allocation (freed on it)
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; o.s = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; o.s = nullptr; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    if (g_alloc_stream) {
      TK_CUDA(cudaMallocAsync(&p, count * sizeof(T), g_alloc_stream));
      s = g_alloc_stream;
    } else {
      TK_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    n = count;
  }
  // grow-only reallocation (contents are not preserved)
  void ensure(size_t count) { if (count > n) alloc(count); }
  void release() {
    if (p) {
      if (s) cudaFreeAsync(p, s);  // ordered after every use on the handle's stream
      else cudaFree(p);
    }
    p = nullptr;
    n = 0;
    s = nullptr;
  }
  size_t bytes() const { return n * sizeof(T); }
};

}  // namespace tk
