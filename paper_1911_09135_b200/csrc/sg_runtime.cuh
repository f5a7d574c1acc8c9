// sg_runtime.cuh — host runtime shared by the BSP drivers (single device:
// sg_engine.cu; edge-cut partitions: sg_dist.cu): kernel launcher (plain /
// CUDA-event profiled), device-resident run buffers, init/advance kernels and
// the push / pull round sequences.
#pragma once
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <unordered_map>

#include "sg_graph.cuh"
#include "sg_bm.cuh"
#include "sg_pull.cuh"

namespace sg {
namespace {

constexpr int64_t kNoHuge = std::numeric_limits<int64_t>::max();

template <class K>
int occupancy_grid(K kernel, int block, int cap_per_sm = 8) {
  static std::mutex mu;
  static std::unordered_map<const void *, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find((const void *)kernel);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0));
  per_sm = std::max(1, std::min(per_sm, cap_per_sm));
  int g = persistent_grid(per_sm);
  cache[(const void *)kernel] = g;
  return g;
}

inline int grid_n(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_info().sms * 32));
}

// Launches round kernels: plain (graph capture) or bracketed by CUDA events.
#ifndef SG_PDL
#define SG_PDL 1
#endif
#ifndef SG_PREFIX_IN_LARGE
#define SG_PREFIX_IN_LARGE 1
#endif
struct Launcher {
  bool profile = false;
  std::vector<std::tuple<const char *, cudaEvent_t, cudaEvent_t>> pending;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, std::pair<int64_t, double>> totals;
  std::vector<std::string> order;

  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    SG_CUDA(cudaEventCreate(&e));
    return e;
  }
  template <class K, class... A>
  void go(const char *name, K kernel, int grid, int block, cudaStream_t s, A... args) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (profile) {
      e0 = ev(), e1 = ev();
      SG_CUDA(cudaEventRecord(e0, s));
    }
    kernel<<<grid, block, 0, s>>>(args...);
    SG_CUDA(cudaGetLastError());
    if (profile) {
      SG_CUDA(cudaEventRecord(e1, s));
      pending.emplace_back(name, e0, e1);
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
  }
  // launch with a programmatic edge to the previous kernel on the stream
  // (the kernel must start with pdl_wait(); see sg_common.cuh)
  template <class K, class... A>
  void go_pdl(const char *name, K kernel, int grid, int block, cudaStream_t s, A... args) {
    if (profile || !SG_PDL) {
      go(name, kernel, grid, block, s, args...);
      return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SG_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  }
  void collect() {
    for (auto &t : pending) {
      float ms = 0;
      SG_CUDA(cudaEventElapsedTime(&ms, std::get<1>(t), std::get<2>(t)));
      std::string n = std::get<0>(t);
      if (!totals.count(n)) order.push_back(n);
      totals[n].first += 1;
      totals[n].second += ms;
      pool.push_back(std::get<1>(t));
      pool.push_back(std::get<2>(t));
    }
    pending.clear();
  }
  ~Launcher() {
    for (auto &t : pending) pool.push_back(std::get<1>(t)), pool.push_back(std::get<2>(t));
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// round context handed to every round body
struct RoundCtx {
  Launcher &L;
  cudaStream_t s;
  cudaGraphConditionalHandle cond;
  int use_cond;
};

// ------------------------------------------------------------ init kernels --
template <class T>
__global__ void k_fill(T *p, int64_t n, T v) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) p[i] = v;
}
template <class T>
__global__ void k_set1(T *p, int64_t i, T v) { p[i] = v; }

__global__ void k_ctl_init(Ctl *ctl, int32_t dense, uint32_t fsize) {
  *ctl = Ctl{};
  ctl->dense = dense;
  ctl->fsize = fsize;
}

__global__ void k_labels_u32(const uint32_t *lab, int64_t n, double *out) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = lab[i] == kInf32 ? INFINITY : (double)lab[i];
}
// u32 labels of the relabeled store -> float64 in the reference's numbering,
// one pass: out[v] = lab[inv[v]] (inv is mostly monotone: the cold vertices
// keep their relative order, so the gather is nearly sequential)
__global__ void k_labels_u32_inv(const uint32_t *__restrict__ lab, const uint32_t *__restrict__ inv,
                                 int64_t n, double *__restrict__ out) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    const uint32_t x = lab[inv[i]];
    out[i] = x == kInf32 ? INFINITY : (double)x;
  }
}
__global__ void k_iota_pairs(uint32_t *p, int64_t n) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    reinterpret_cast<uint2 *>(p)[i] = make_uint2((uint32_t)i, (uint32_t)i);
}
__global__ void k_labels_f64bits(const unsigned long long *lab, int64_t n, double *out) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = __longlong_as_double((long long)lab[i]);
}
__global__ void k_iota(uint32_t *p, int64_t n) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    p[i] = (uint32_t)i;
}
// after R rounds the half written last, R & 1, holds every final label
__global__ void k_labels_pair_u32(const uint32_t *lab, int64_t n, const Ctl *ctl, double *out) {
  const uint32_t h = ctl->round & 1;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    uint32_t x = lab[2 * i + h];
    out[i] = x == kInf32 ? INFINITY : (double)x;
  }
}
__global__ void k_labels_pair_f64(const unsigned long long *lab, int64_t n, const Ctl *ctl,
                                  double *out) {
  const uint32_t h = ctl->round & 1;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = __longlong_as_double((long long)lab[2 * i + h]);
}
__global__ void k_labels_alive(const uint8_t *a, int64_t n, double *out) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = a[i] ? 1.0 : 0.0;
}

// inv_outdeg (apps.py:158-161), rank_0 = 1-d and round-0 aux = rank*inv (apps.py:162,176)
__global__ void k_pr_init(const int64_t *off, int64_t n, double omd, double *inv, double *rank,
                          double *aux) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += st) {
    int64_t d = off[v + 1] - off[v];
    double iv = d > 0 ? 1.0 / (double)d : 0.0;
    inv[v] = iv;
    rank[v] = omd;
    aux[v] = __dmul_rn(omd, iv);
  }
}
// gain[v] = sum_{u->v} inv[u] (apps.py:166-168), max over v by atomicMax.
// Rows up to kGainThread edges: one thread folds its row left to right in
// CSC (== CSR edge) order, exactly as np.bincount accumulates it.  Longer rows
// (the hubs, where the maximum usually is): one warp, strided partial sums and
// a tree reduction -- the same value to within rounding (a few ulp), which only
// matters if a round's max|delta| lands within those ulps of eps_stop.
constexpr int64_t kGainThread = 64;
__global__ void k_pr_gain_rows(const int64_t *off, const uint32_t *col, int64_t n,
                               const double *inv, unsigned long long *maxbits) {
  double best = 0.0;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += st) {
    const int64_t b = off[v], e = off[v + 1];
    if (e - b > kGainThread) continue;
    double acc = 0.0;
    for (int64_t j = b; j < e; j += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = j + u < e ? inv[col[j + u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u < e) acc = __dadd_rn(acc, x[u]);
    }
    best = acc > best ? acc : best;
  }
  best = warp_max(best);
  if (lane_id() == 0 && best > 0)
    atomicMax(maxbits, (unsigned long long)__double_as_longlong(best));
}
constexpr int64_t kGainWarp = 8192;  // longer rows: one CTA each (k_pr_gain_big)
__global__ void k_pr_gain_max(const int64_t *off, const uint32_t *col, int64_t n,
                              const double *inv, unsigned long long *maxbits, uint32_t *big,
                              uint32_t *nbig) {
  int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double best = 0.0;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const int64_t b = off[v], e = off[v + 1];
    if (e - b <= kGainThread) continue;
    if (e - b > kGainWarp) {
      if (lane_id() == 0) big[atomicAdd(nbig, 1u)] = (uint32_t)v;
      continue;
    }
    double acc = 0.0;
    for (int64_t j = b + lane_id(); j < e; j += 32 * 4) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = j + 32 * u < e ? inv[col[j + 32 * u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += x[u];
    }
    acc = warp_sum(acc);
    best = acc > best ? acc : best;
  }
  if (lane_id() == 0 && best > 0)
    atomicMax(maxbits, (unsigned long long)__double_as_longlong(best));
}

__global__ void __launch_bounds__(256) k_pr_gain_big(const int64_t *off, const uint32_t *col,
                                                     const double *inv, const uint32_t *big,
                                                     const uint32_t *nbig,
                                                     unsigned long long *maxbits) {
  __shared__ double red[32];
  for (uint32_t i = blockIdx.x; i < *nbig; i += gridDim.x) {
    const uint32_t v = big[i];
    const int64_t b = off[v], e = off[v + 1];
    double acc = 0.0;
    for (int64_t j = b + threadIdx.x; j < e; j += 256 * 4) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = j + 256 * u < e ? inv[col[j + 256 * u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += x[u];
    }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0 && acc > 0)
      atomicMax(maxbits, (unsigned long long)__double_as_longlong(acc));
    __syncthreads();
  }
}

// static bins of a dense pull view (pr): CTA-bin rows and huge rows
__global__ void k_static_bins(const int64_t *off, uint32_t lo, uint32_t n, int64_t thr,
                              uint32_t *largeq, uint32_t *hugeq, Ctl *ctl, Cuts cuts) {
  uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long le = 0;
  uint32_t lbm = 0;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < n; b += st) {
    const bool in = b + threadIdx.x < n;
    uint64_t v = lo + b + threadIdx.x;
    int64_t d = in ? off[v + 1] - off[v] : 0;
    bool huge = in && d >= thr;
    bool large = in && !huge && d >= (int64_t)kLarge;
    if (large) le += (unsigned long long)d;
    if (huge && cuts.D > 1) lbm |= 1u << owner_of(cuts, (uint32_t)v);
    warp_append(huge, (uint32_t)v, hugeq, &ctl->nhuge);
    warp_append(large, (uint32_t)v, largeq, &ctl->nlarge);
  }
  le = warp_sum(le);
  lbm = __reduce_or_sync(kFull, lbm);
  if (lane_id() == 0 && le) atomicAdd(&ctl->large_edges, le);
  if (lane_id() == 0 && lbm) atomicOr(&ctl->part_lb_mask, lbm);
}

// ------------------------------------------------- edge-cut partitioning --
// make_partition (engine.py:64-85): cut_k = searchsorted(off, round(k*E/D), 'left'),
// kept monotone; Python's round() is round-half-even == rint() by default.
__global__ void k_cuts(const int64_t *off, int64_t nv, int D, long long *cuts) {
  if (threadIdx.x || blockIdx.x) return;
  const long long E = off[nv];
  cuts[0] = 0;
  for (int k = 1; k < D; ++k) {
    const long long target = (long long)rint((double)((long long)k * E) / (double)D);
    int64_t lo = 0, hi = nv + 1;  // first i with off[i] >= target
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (off[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    cuts[k] = lo > cuts[k - 1] ? lo : cuts[k - 1];
  }
  cuts[D] = nv;
}
// mirror_count[v] = #partitions (other than v's owner) whose rows point at v
__global__ void k_mirror_bits(const int64_t *off, const uint32_t *col, int64_t nv, Cuts cuts,
                              uint32_t *bits) {
  int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nv; u += warps) {
    const int d = owner_of(cuts, (uint32_t)u);
    const uint32_t bit = 1u << d;
    for (int64_t e = off[u] + lane_id(); e < off[u + 1]; e += 32) {
      const uint32_t t = col[e];
      if ((t < cuts.c[d] || t >= cuts.c[d + 1]) && !(bits[t] & bit)) atomicOr(bits + t, bit);
    }
  }
}
__global__ void k_popc(uint32_t *bits, int64_t n) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    bits[i] = __popc(bits[i]);
}

inline Cuts make_cuts(const View &v, int D) {
  if (D < 1 || D > kMaxParts)
    throw Error(SG_ECONFIG, "devices must be in [1, " + std::to_string(kMaxParts) + "]");
  Cuts c{};
  c.D = D;
  c.c[0] = 0, c.c[1] = v.nv;
  if (D == 1) return c;
  DBuf<long long> d(D + 1);
  k_cuts<<<1, 1>>>(v.off.p, v.nv, D, d.p);
  SG_CUDA(cudaGetLastError());
  SG_CUDA(cudaMemcpy(c.c, d.p, sizeof(long long) * (D + 1), cudaMemcpyDeviceToHost));
  return c;
}
inline void mirror_counts(const View &v, const Cuts &c, uint32_t *mc) {
  SG_CUDA(cudaMemset(mc, 0, sizeof(uint32_t) * std::max<int64_t>(v.nv, 1)));
  k_mirror_bits<<<grid_n(v.nv * 32), 256>>>(v.off.p, v.col.p, v.nv, c, mc);
  SG_CUDA(cudaGetLastError());
  k_popc<<<grid_n(v.nv), 256>>>(mc, v.nv);
  SG_CUDA(cudaGetLastError());
  SG_CUDA(cudaDeviceSynchronize());
}

// ------------------------------------------------------- advance kernels --
struct Loop {
  int64_t limit, max_rounds;
  cudaGraphConditionalHandle cond;
  int use_cond;
};

__device__ __forceinline__ void loop_test(Ctl *ctl, uint32_t round, bool empty, const Loop &lp) {
  if (empty) ctl->done = 1;
  else if ((int64_t)round + 1 >= lp.limit)
    ctl->error = (int64_t)round + 1 >= lp.max_rounds ? SG_ECONVERGE : SG_ENOMEM, ctl->done = 1;
  if (lp.use_cond) cudaGraphSetConditional(lp.cond, ctl->done ? 0u : 1u);
}

// round bookkeeping (the parity-paired labels need no commit pass)
__device__ __forceinline__ void push_advance(const PushArgs &a, const Loop &lp);
__global__ void k_push_advance(PushArgs a, Loop lp) {
  pdl_wait();
  pdl_trigger();
  push_advance(a, lp);
}
// the same outside the round graph (no programmatic-launch edge to what follows)
__global__ void k_push_advance_plain(PushArgs a, Loop lp) { push_advance(a, lp); }
__device__ __forceinline__ void push_advance(const PushArgs &a, const Loop &lp) {
  Ctl *ctl = a.ctl;
  if (threadIdx.x) return;
  if (ctl->done) {
    if (lp.use_cond) cudaGraphSetConditional(lp.cond, 0u);
    return;
  }
  const uint32_t round = ctl->round;
  const uint32_t nn = ctl->nsize, nz = ctl->nzero;
  RoundStat &s = a.stats[round];
  s.frontier_size = ctl->dense ? a.nv : ctl->fsize + ctl->fzero;
  s.active_edges = (long long)ctl->edges;
  s.huge_count = ctl->nhuge;
  s.huge_edges = (long long)ctl->huge_edges;
  s.large_count = ctl->nlarge;
  s.large_edges = (long long)ctl->large_edges;
  s.updated = (long long)nn + nz;
  s.comm_sent = (long long)ctl->comm_sent;
  s.comm_broadcast = (long long)ctl->comm_bcast;
  // alb / twc: inspect + twc per non-empty round, lb when huge vertices exist;
  // lb: one lb launch when the prefix has edges (schedulers.py:280-283);
  // vertex / edge: one launch per non-empty round (reported as launches_twc)
  s.launches_twc = a.sched == 1 ? 0 : s.frontier_size > 0;
  s.launches_lb = a.sched == 1 ? ctl->huge_edges > 0 : a.sched == 0 ? ctl->nhuge > 0 : 0;
  if (a.sched >= 2) s.huge_count = s.large_count = s.large_edges = 0, s.huge_edges = 0;
  ctl->fsize = nn;
  ctl->fzero = nz;
  ctl->nsize = 0;
  ctl->nzero = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = ctl->chunk_head = 0;
  ctl->edges = ctl->huge_edges = ctl->large_edges = ctl->comm_sent = ctl->comm_bcast = 0;
  ctl->dense = 0;
  ctl->ticket = 0;
  ctl->round = round + 1;
  loop_test(ctl, round, nn == 0 && nz == 0, lp);
  __threadfence();
}

// kcore: kill the dying (apps.py:225); devices > 1: their mirrors get the broadcast
__global__ void k_kcore_kill(PullArgs a, uint8_t *alive) {
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t nd = ctl->ndying;
  unsigned long long b = 0;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += st) {
    const uint32_t v = a.dying[i];
    alive[v] = 0;
    if (a.mcount) b += a.mcount[v];
  }
  b = warp_sum(b);
  if (lane_id() == 0 && b) atomicAdd(&ctl->comm_bcast, b);
}
// record the count-phase stats; the neighbour walk then reuses the CTA-bin queue
__global__ void k_kcore_reset(PullArgs a) {
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  RoundStat &s = a.stats[ctl->round];
  s.frontier_size = ctl->dense ? a.nv : ctl->fsize;
  s.active_edges = (long long)ctl->edges;
  s.huge_count = ctl->nhuge;
  s.huge_edges = (long long)ctl->huge_edges;
  s.large_count = ctl->nlarge;
  s.large_edges = (long long)ctl->large_edges;
  s.updated = (long long)ctl->ndying + ctl->fzero;
  s.comm_sent = 0;
  s.comm_broadcast = (long long)ctl->comm_bcast;
  s.launches_twc = a.cuts.D > 1 ? __popc(ctl->part_twc_mask) : s.frontier_size > 0;
  s.launches_lb = a.cuts.D > 1 ? __popc(ctl->part_lb_mask) : ctl->nhuge > 0;
  ctl->comm_bcast = 0;
  ctl->part_twc_mask = ctl->part_lb_mask = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = ctl->chunk_head = 0;
  ctl->huge_edges = ctl->large_edges = 0;
}

__global__ void k_kcore_advance(Ctl *ctl, Loop lp) {
  if (ctl->done) {
    if (lp.use_cond) cudaGraphSetConditional(lp.cond, 0u);
    return;
  }
  const uint32_t round = ctl->round;
  const uint32_t nd = ctl->ndying + ctl->fzero, nn = ctl->nsize;
  ctl->fsize = nn;
  ctl->fzero = 0;
  ctl->nsize = 0;
  ctl->ndying = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = ctl->chunk_head = 0;
  ctl->edges = ctl->huge_edges = ctl->large_edges = 0;
  ctl->dense = 0;
  ctl->round = round + 1;
  loop_test(ctl, round, nd == 0 || nn == 0, lp);  // apps.py:223-232
}

// ------------------------------------------------------------ run state --
// Device round-log capacity of a run: min(max_rounds, 2^20) records first; a
// run that outgrows it is repeated with room for max_rounds (up to 2^26
// records, 5.9 GB), so the only round limit is the reference's max_rounds
// (engine.py:206-209).  Runs are deterministic, so the repeat is identical.
inline int64_t &stats_cap_limit() {
  static thread_local int64_t lim = (int64_t)1 << 20;
  return lim;
}
inline int64_t stats_cap(int64_t max_rounds) {
  return std::max<int64_t>(1, std::min<int64_t>(max_rounds, stats_cap_limit()));
}
constexpr int64_t kStatsCapMax = (int64_t)1 << 26;

struct RunBufs {
  DBuf<Ctl> ctl;
  DBuf<RoundStat> stats;
  int64_t stats_cap = 0;
  DBuf<uint32_t> q0, q1, largeq, hugeq, dying;
  DBuf<int64_t> hpre, hstart;
  DBuf<unsigned long long> hval, largesv;
  // SG_FLAG_CTA_COUNTS: per-CTA processed edges of the first cta_rounds rounds
  bool want_cta = false;
  DBuf<unsigned long long> cta;
  uint32_t cta_g = 0, cta_rounds = 0;

  void alloc_common(int64_t nv, int64_t rounds_cap) {
    size_t n = (size_t)std::max<int64_t>(nv, 1);
    if (want_cta) {
      cta_g = (uint32_t)sm_info().sms;  // one slot per SM
      cta_rounds = (uint32_t)std::min<int64_t>(rounds_cap, 4096);
      cta.alloc((size_t)cta_g * cta_rounds);
    }
    // no memset here: every driver zeroes the block with k_ctl_init on its own
    // (non-blocking) stream; a legacy-stream memset is NOT ordered before that
    // and could land after it (seen as a lost dense frontier with ranks as threads)
    ctl.alloc(1);
    stats_cap = rounds_cap;
    stats.alloc(rounds_cap);
    q0.alloc(n), q1.alloc(n), largeq.alloc(n), hugeq.alloc(n);
    hpre.alloc(n), hstart.alloc(n), hval.alloc(n), largesv.alloc(n);
  }
  PushArgs push_args(const View &v, int64_t thr) {
    PushArgs a{};
    a.off = v.off.p;
    a.col = v.col.p;
    a.nv = (uint32_t)v.nv;
    a.ctl = ctl.p;
    a.q[0] = q0.p, a.q[1] = q1.p;
    a.largeq = largeq.p, a.hugeq = hugeq.p;
    a.hpre = hpre.p, a.hstart = hstart.p, a.hval = hval.p;
    a.largesv = largesv.p;
    a.dying = dying.p;
    a.threshold = thr;
    a.src_mode = 0;
    a.stats = stats.p;
    a.no_enqueue = 0;
    a.dense_lo = 0;
    a.dense_n = (uint32_t)v.nv;
    a.cta_edges = cta.p, a.cta_g = cta_g, a.cta_rounds = cta_rounds;
    return a;
  }
  PullArgs pull_args(const View &v, int64_t thr, int dyn) {
    PullArgs a{};
    a.off = v.off.p;
    a.col = v.col.p;
    a.nv = (uint32_t)v.nv;
    a.ctl = ctl.p;
    a.q[0] = q0.p, a.q[1] = q1.p;
    a.largeq = largeq.p, a.hugeq = hugeq.p;
    a.hpre = hpre.p, a.hstart = hstart.p;
    a.threshold = thr;
    a.dynamic_bins = dyn;
    a.dying = dying.p;
    a.stats = stats.p;
    a.row_lo = 0;
    a.row_n = (uint32_t)v.nv;
    a.cta_edges = cta.p, a.cta_g = cta_g, a.cta_rounds = cta_rounds;
    return a;
  }
};

// A prepared run: buffers allocated, nothing launched yet.
struct Program {
  std::function<void(Launcher &, cudaStream_t)> init;  // device state init (timed)
  std::function<void(RoundCtx &)> round;              // one BSP round
  std::function<void(Launcher &, cudaStream_t)> finish;  // labels -> out (untimed)
  // relabeled store: a finish that maps the labels back to the reference's
  // numbering itself (gathering through `inv` into `out`) sets `unpermuted`
  const uint32_t *inv = nullptr;
  double *out = nullptr;
  bool unpermuted = false;
  std::vector<std::shared_ptr<void>> keep;
  template <class T>
  T *buf(int64_t n) {
    auto b = std::make_shared<DBuf<T>>(std::max<int64_t>(n, 1));
    keep.push_back(b);
    return b->p;
  }
};

template <class T>
void fill(Launcher &L, T *p, int64_t n, T v, cudaStream_t s) {
  if (n > 0) L.go("init", k_fill<T>, grid_n(n), 256, s, p, n, v);
}

// ----------------------------------------------------------------- apps --
template <class Op>
void push_round(RoundCtx &c, const PushArgs &a, const Op &op, bool blocked) {
  c.L.go("push_twc", k_push_twc<Op>, occupancy_grid(k_push_twc<Op>, kTB), kTB, c.s, a, op);
  c.L.go("push_large", k_push_large<Op>, occupancy_grid(k_push_large<Op>, kTB), kTB, c.s, a, op);
  if (a.threshold != kNoHuge) {
    c.L.go("huge_prefix", k_huge_prefix<Op>, 1, 1024, c.s, a, op);
    if (blocked)
      c.L.go("push_lb", k_push_lb<Op, true>, occupancy_grid(k_push_lb<Op, true>, kTB), kTB, c.s, a,
             op);
    else
      c.L.go("push_lb", k_push_lb<Op, false>, occupancy_grid(k_push_lb<Op, false>, kTB), kTB, c.s,
             a, op);
  }
}

#ifndef SG_LARGE_VEC
#define SG_LARGE_VEC 0  // 1: CTA bin with 128-bit adjacency loads (k_bm_large_vec)
#endif
#ifndef SG_LARGE_STAGE
#define SG_LARGE_STAGE 0  // 1: CTA bin with cp.async-staged adjacency (k_bm_large_staged)
#endif
#ifndef SG_LARGE_PIPE
#define SG_LARGE_PIPE 1
#endif
// single-device push round with the bitmap next-frontier (sg_bm.cuh)
template <class Op>
void bm_round(RoundCtx &c, const PushArgs &a, const Op &op, bool blocked, bool classic = false,
              long long *tsum = nullptr, bool compact = true) {
  if (a.sched == 2) {  // vertex
    c.L.go("push_vertex", k_bm_vertex<Op>, occupancy_grid(k_bm_vertex<Op>, kTB), kTB, c.s, a, op);
    if (compact)
      c.L.go("compact", k_bm_compact<Op>, occupancy_grid(k_bm_compact<Op>, kTB), kTB, c.s, a, op);
    return;
  }
  if (a.sched == 1 || a.sched == 3) {  // lb / edge: prefix over the whole frontier
    const int g = occupancy_grid(k_front_tiles<Op>, kTB);
    c.L.go("front_prefix", k_front_tiles<Op>, g, kTB, c.s, a, op, tsum);
    c.L.go("front_prefix", k_front_scan, 1, 1024, c.s, a, tsum);
    c.L.go("front_prefix", k_front_apply, g, kTB, c.s, a, (const long long *)tsum);
    if (a.sched == 3)
      c.L.go("push_edge", k_bm_edge<Op>, occupancy_grid(k_bm_edge<Op>, kTB), kTB, c.s, a, op);
    else if (blocked)
      c.L.go("push_lb", k_bm_lb<Op, true>, occupancy_grid(k_bm_lb<Op, true>, kTB), kTB, c.s, a, op);
    else
      c.L.go("push_lb", k_bm_lb<Op, false>, occupancy_grid(k_bm_lb<Op, false>, kTB), kTB, c.s, a,
             op);
    if (compact)
      c.L.go("compact", k_bm_compact<Op>, occupancy_grid(k_bm_compact<Op>, kTB), kTB, c.s, a, op);
    return;
  }
  // the huge prefix is built by the CTA-bin kernel's CTA 0 (one node fewer)
  PushArgs a2 = a;
  a2.prefix_in_large = SG_PREFIX_IN_LARGE && a.threshold != kNoHuge;
  c.L.go_pdl("push_twc", k_bm_twc<Op>, occupancy_grid(k_bm_twc<Op>, kTB), kTB, c.s, a, op);
  if (classic)
    c.L.go_pdl("push_large", k_bm_large_classic<Op>, occupancy_grid(k_bm_large_classic<Op>, kTB), kTB,
           c.s, a2, op);
  else if (SG_LARGE_VEC && !std::is_same<typename Op::W, int64_t>::value)
    c.L.go_pdl("push_large", k_bm_large_vec<Op>, occupancy_grid(k_bm_large_vec<Op>, kTB), kTB,
               c.s, a2, op);
  else if (SG_LARGE_STAGE && !std::is_same<typename Op::W, int64_t>::value)
    c.L.go_pdl("push_large", k_bm_large_staged<Op>, occupancy_grid(k_bm_large_staged<Op>, kTB),
               kTB, c.s, a2, op);
  else if (SG_LARGE_PIPE)
    c.L.go_pdl("push_large", k_bm_large_pipe<Op>, occupancy_grid(k_bm_large_pipe<Op>, kTB), kTB, c.s,
           a2, op);
  else
    c.L.go_pdl("push_large", k_bm_large<Op>, occupancy_grid(k_bm_large<Op>, kTB), kTB, c.s, a2, op);
  if (a.threshold != kNoHuge) {
    if (!a2.prefix_in_large) c.L.go_pdl("huge_prefix", k_huge_prefix<Op>, 1, 1024, c.s, a, op);
    if (blocked)
      c.L.go_pdl("push_lb", k_bm_lb<Op, true>, occupancy_grid(k_bm_lb<Op, true>, kTB), kTB, c.s, a, op);
    else
      c.L.go_pdl("push_lb", k_bm_lb<Op, false>, occupancy_grid(k_bm_lb<Op, false>, kTB), kTB, c.s, a,
             op);
  }
  if (compact)
    c.L.go_pdl("compact", k_bm_compact<Op>, occupancy_grid(k_bm_compact<Op>, kTB), kTB, c.s, a, op);
}

template <class Op>
void pull_round(RoundCtx &c, const PullArgs &a, const Op &op, bool blocked, typename Op::A *hacc,
                bool classic = false) {
  if (a.vertex) {  // vertex scheduler: one thread per row
    c.L.go("pull_vertex", k_pull_vertex<Op>, occupancy_grid(k_pull_vertex<Op>, kTB), kTB, c.s, a,
           op);
    return;
  }
  c.L.go("pull_twc", k_pull_twc<Op>, occupancy_grid(k_pull_twc<Op>, kTB), kTB, c.s, a, op);
  if (classic)
    c.L.go("pull_large", k_pull_large_classic<Op>, occupancy_grid(k_pull_large_classic<Op>, kTB),
           kTB, c.s, a, op);
  else
    c.L.go("pull_large", k_pull_large<Op>, occupancy_grid(k_pull_large<Op>, kTB), kTB, c.s, a, op);
  if (a.threshold != kNoHuge) {
    if (a.dynamic_bins) c.L.go("huge_prefix", k_pull_prefix, 1, 1024, c.s, a);
    if (blocked)
      c.L.go("pull_lb", k_pull_lb<Op, true>, occupancy_grid(k_pull_lb<Op, true>, kTB), kTB, c.s, a,
             op, hacc);
    else
      c.L.go("pull_lb", k_pull_lb<Op, false>, occupancy_grid(k_pull_lb<Op, false>, kTB), kTB, c.s,
             a, op, hacc);
  }
}

Loop loop_of(const RunBufs &rb, int64_t max_rounds, const RoundCtx &c) {
  return Loop{std::min<int64_t>(max_rounds, rb.stats_cap), max_rounds, c.cond, c.use_cond};
}


}  // namespace
}  // namespace sg
