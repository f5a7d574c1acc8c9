// sg_common.cuh — shared host/device plumbing for libsimtgraph_cuda (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/simtgraph_cuda.h"

namespace sg {

constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kInf32 = 0xffffffffu;  // +inf for u32 labels (bfs hops, cc ids, sssp sums)

// ---------------------------------------------------------------- errors --
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);
extern std::atomic<int64_t> g_launches;

#define SG_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::sg::Error(e_ == cudaErrorMemoryAllocation ? SG_ENOMEM : SG_ECUDA,           \
                        std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +       \
                            __FILE__ + ":" + std::to_string(__LINE__));                   \
  } while (0)

// launch + count + check (async errors surface at the next sync)
#define SG_LAUNCH(kernel, grid, block, smem, stream, ...)                                 \
  do {                                                                                    \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                           \
    ::sg::g_launches.fetch_add(1, std::memory_order_relaxed);                             \
    SG_CUDA(cudaGetLastError());                                                          \
  } while (0)

template <class F>
int guard(F &&f) {
  try {
    f();
    return SG_OK;
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc &) {
    set_last_error("host allocation failed");
    return SG_ENOMEM;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SG_ECUDA;
  }
}

// --------------------------------------------------------- device buffer --
// Caching device allocator (sg_engine.cu): freed blocks are kept per size and
// reused, so repeated graph uploads and runs do not pay cudaMalloc / cudaFree
// (each a device-wide synchronisation).  Contract: a block is released only
// after the stream work that uses it has completed (every driver synchronises
// its stream before its buffers go out of scope).  On allocation failure the
// cache is returned to the driver and the allocation retried.
void *dev_alloc(size_t bytes);
void dev_free(void *p);
void dev_release_cached();
void *host_alloc(size_t bytes);  // pinned, cached (result buffers)
void host_free(void *p);

template <class T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T *>(dev_alloc(sizeof(T) * count));
  }
  void release() {
    if (p) dev_free(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return sizeof(T) * n; }
  T *get() const { return p; }
};

struct SmInfo {
  int sms = 148;
  int device = 0;
};
const SmInfo &sm_info();

// persistent grid: `per_sm` resident CTAs on every SM
inline int persistent_grid(int per_sm) { return sm_info().sms * per_sm; }

// ------------------------------------------------------------ warp utils --
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
// Programmatic dependent launch (sm_90+): the per-round kernels of the push
// loop are launched with programmatic stream serialization, so a kernel's CTAs
// are scheduled while its predecessor drains; every such kernel waits for the
// predecessor's completion (and memory) before its first access, and lets its
// own successor launch right away.  Without a programmatic edge both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class T>
__device__ __forceinline__ T warp_incl_scan(T x) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = __shfl_up_sync(kFull, x, d);
    if (lane_id() >= (uint32_t)d) x += y;
  }
  return x;
}

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
  return x;
}

template <class T>
__device__ __forceinline__ T warp_max(T x) {
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    T y = __shfl_xor_sync(kFull, x, d);
    x = y > x ? y : x;
  }
  return x;
}

// streaming (read-once) loads: keep the adjacency / weights out of L1 and mark
// them evict-first in L2, so the L2 holds the randomly accessed labels instead
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(l2_evict_first()));
  return v;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t *p) {
  long long v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;"
               : "=l"(v)
               : "l"(p), "l"(l2_evict_first()));
  return v;
}
// label reads that must not hit a stale L1 line of an earlier round (L2 only)
__device__ __forceinline__ uint32_t ld_l2(const uint32_t *p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_l2(const unsigned long long *p) {
  return __ldcg(p);
}

}  // namespace sg
