// sg_ctl.cuh — device-resident BSP round control.
//
// Every kernel of a round reads the round index, frontier size and done flag
// from this block, so a round is a fixed sequence of launches with fixed
// arguments (capturable in a CUDA graph) and the host never has to read a
// count to launch the next round (it checks `done` every few rounds).
#pragma once
#include "sg_common.cuh"

namespace sg {

struct Ctl {
  int32_t round;        // index of the round being executed (engine.py:205 loop count)
  int32_t done;         // frontier empty / pr converged / error
  int32_t error;        // SG_ECONVERGE when max_rounds is exceeded (engine.py:206-209)
  int32_t dense;        // current frontier is all of [0, nv) (cc / kcore round 0, pr)
  uint32_t fsize;       // current frontier size (queue q[round & 1])
  uint32_t nsize;       // next-frontier enqueue cursor (queue q[(round + 1) & 1])
  uint32_t nlarge;      // CTA-bin vertices found by inspection this round
  uint32_t nhuge;       // huge vertices found by inspection this round
  uint32_t large_head;  // dynamic fetch cursor of the CTA-bin kernel
  uint32_t ticket;      // last-block ticket of the advance kernels
  uint32_t ndying;      // kcore: vertices whose count fell below k this round
  uint32_t chunk_head;  // dynamic fetch cursor of the TWC kernel (units of kChunkGrab warps)
  unsigned long long edges;       // active edges (sum of frontier degrees) this round
  unsigned long long huge_edges;  // PrefixWork.total_edges
  unsigned long long delta_bits;  // pr: max |new - old| (double bits, >= 0)
  unsigned long long comm_sent;
  unsigned long long comm_bcast;
  unsigned long long large_edges;  // edges of CTA-bin vertices this round
  // relabeled store: frontier members with no out-edges (ids >= PushArgs::zlo)
  // are counted, not queued -- current frontier / next frontier
  uint32_t fzero, nzero;
  uint32_t part_twc_mask;  // devices>1 accounting: partitions with a non-empty local frontier
  uint32_t part_lb_mask;   // ... whose local frontier holds a huge vertex
};

// Edge-cut partition of a traversal view (engine.py:64-85): partition d owns
// rows [c[d], c[d+1]).  D == 1 disables the per-partition accounting.
constexpr int kMaxParts = 32;
struct Cuts {
  long long c[kMaxParts + 1];
  int D;
};
__device__ __forceinline__ int owner_of(const Cuts &k, uint32_t v) {
  int d = 0;
  while (d + 1 < k.D && (long long)v >= k.c[d + 1]) ++d;
  return d;
}

// Dynamic work fetch of the persistent grids: a unit's (warp's / CTA's) first
// grab is its own index, only later grabs go through the round's shared
// counter (offset by the number of units).  At a small frontier most of a
// 740-CTA grid then exits without touching the counter: thousands of warps
// serialising on one atomic cost ~10-15 us per launch.
constexpr uint32_t kNoGrab = 0xffffffffu;
__device__ __forceinline__ uint32_t global_warp() {
  return (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ uint32_t grid_warps() { return (gridDim.x * blockDim.x) >> 5; }
__device__ __forceinline__ uint32_t cta_grab(uint32_t *ctr, bool &first) {
  if (first) {
    first = false;
    return blockIdx.x;
  }
  return atomicAdd(ctr, 1u) + gridDim.x;
}

// one record per round, layout == sg_round (include/simtgraph_cuda.h)
struct RoundStat {
  long long frontier_size, active_edges, huge_count, huge_edges, large_count, large_edges,
      updated, comm_sent, comm_broadcast, launches_twc, launches_lb;
};
static_assert(sizeof(RoundStat) == sizeof(sg_round), "RoundStat must mirror sg_round");

// Per-warp staging of enqueued vertex ids in shared memory: one global
// atomic per ~224 ids and coalesced copies out, instead of one contended
// atomic per warp per edge chunk.
constexpr int kWQ = 256;
struct WarpQueue {
  uint32_t *buf;  // kWQ shared-memory slots owned by this warp
  uint32_t n;     // warp-uniform fill level
  uint32_t *gq;
  uint32_t *gcount;

  __device__ __forceinline__ void flush() {
    if (!gq) return;
    __syncwarp();
    uint32_t base = 0;
    if (lane_id() == 0 && n) base = atomicAdd(gcount, n);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t j = lane_id(); j < n; j += 32) gq[base + j] = buf[j];
    __syncwarp();
    n = 0;
  }
  // must be called by all 32 lanes (converged); a null queue discards (partitioned
  // runs rebuild frontiers from the exchanged labels instead)
  __device__ __forceinline__ void push(bool p, uint32_t v) {
    if (!gq) return;
    uint32_t m = __ballot_sync(kFull, p);
    if (!m) return;
    if (p) buf[n + __popc(m & lanemask_lt())] = v;
    n += __popc(m);
    if (n > kWQ - 32) flush();
  }
};

// warp-aggregated append of flagged lanes to a global list (rare events);
// returns each flagged lane's slot
__device__ __forceinline__ uint32_t warp_append(bool p, uint32_t v, uint32_t *list,
                                                uint32_t *count) {
  uint32_t m = __ballot_sync(kFull, p);
  if (!m) return 0;
  uint32_t base = 0;
  if (lane_id() == (uint32_t)(__ffs(m) - 1)) base = atomicAdd(count, (uint32_t)__popc(m));
  base = __shfl_sync(kFull, base, __ffs(m) - 1);
  const uint32_t slot = base + __popc(m & lanemask_lt());
  if (p) list[slot] = v;
  return slot;
}

template <class T>
__device__ __forceinline__ T block_sum(T x, T *smem /* >= 32 */) {
  x = warp_sum(x);
  __syncthreads();
  if (lane_id() == 0) smem[threadIdx.x >> 5] = x;
  __syncthreads();
  T r = 0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? smem[threadIdx.x] : T(0);
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// first lane o of a warp whose inclusive prefix exceeds `slot` (prefixes non-decreasing)
__device__ __forceinline__ int warp_owner(uint32_t incl, uint32_t slot) {
  int o = 0;
#pragma unroll
  for (int step = 16; step; step >>= 1) {
    uint32_t iv = __shfl_sync(kFull, incl, o + step - 1);
    if (iv <= slot) o += step;
  }
  return o;
}

__device__ __forceinline__ int64_t shfl64(int64_t x, int src) {
  return (int64_t)__shfl_sync(kFull, (long long)x, src);
}

// upper_bound: first i in [0, n) with pre[i] > g (pre inclusive, increasing)
__device__ __forceinline__ uint32_t owner_search(const int64_t *pre, uint32_t n, int64_t g) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (g < pre[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Two-level find_owner for the LB kernels' chunk bisection: a shared-memory
// sample of the huge prefix (every stride-th block end, <= kCoarse entries)
// narrows the search to one stride-long block before the global-memory steps
// (cc rmat24 round 0: 2,325 hubs -> 8 shared + 4 global steps instead of 11
// global ones); 2 KB of shared memory, so the L1 keeps its size.
constexpr uint32_t kCoarse = 256;
struct Coarse {
  const int64_t *pre;  // the inclusive huge prefix (global)
  const int64_t *c;    // c[j] = pre[min((j + 1) * stride, n) - 1] (shared)
  uint32_t n, stride, m;
  // upper_bound: first i with pre[i] > g (g < pre[n - 1])
  __device__ __forceinline__ uint32_t find(int64_t g) const {
    uint32_t lo = 0, hi = m - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (g < c[mid]) hi = mid;
      else lo = mid + 1;
    }
    uint32_t a = lo * stride, b = min(a + stride, n) - 1;
    while (a < b) {
      const uint32_t mid = (a + b) >> 1;
      if (g < pre[mid]) b = mid;
      else a = mid + 1;
    }
    return a;
  }
};
// all threads of the CTA: fill the sample (c has kCoarse entries)
__device__ __forceinline__ Coarse coarse_build(int64_t *c, const int64_t *pre, uint32_t n) {
  Coarse x{pre, c, n, (n + kCoarse - 1) / kCoarse, 0};
  x.m = (n + x.stride - 1) / x.stride;
  for (uint32_t i = threadIdx.x; i < x.m; i += blockDim.x) c[i] = pre[min((i + 1) * x.stride, n) - 1];
  __syncthreads();
  return x;
}

}  // namespace sg
