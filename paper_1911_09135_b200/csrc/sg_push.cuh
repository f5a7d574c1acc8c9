// sg_push.cuh — ALB push round: inspection + TWC bins + huge-vertex LB kernel.
//
// Reference semantics (schedulers.py:252-298, _kernels_py.py:69-85/120-201):
//   inspect   : deg(v) for every active v; huge = deg >= t; the rest go to
//               TWC bins (small < W <= medium < threads_per_cta <= large)
//   LB kernel : the edges of all huge vertices, numbered g in [0, e) through
//               the inclusive prefix of their degrees, distributed cyclically
//               (g = p*T + tid) or blocked over every thread of every CTA;
//               the owner of g is found by binary search over the prefix
//   operator  : prop = values[row] (+1 | +w | +0); out[dst] = min(out[dst], prop)
// B200 mapping:
//   * inspection is fused into the TWC kernel: each warp reads 32 frontier ids,
//     their offsets and snapshot labels; huge / CTA-bin vertices are appended to
//     device queues, the small+medium vertices of the warp are processed right
//     there by warp-level scan-based gathering (Merrill's fine-grained TWC: the
//     warp's edges are numbered by a shuffle scan and lanes take consecutive
//     edge slots, so adjacency loads are coalesced);
//   * CTA bin: one CTA per vertex (dynamic fetch), 256 consecutive edges per step;
//   * huge bin: a single-CTA scan builds the int64 prefix + snapshot labels, the
//     LB kernel stages the prefix in shared memory and every thread of every CTA
//     walks g cyclically: consecutive lanes read consecutive adjacency entries;
//   * BSP: sources read the round-start snapshot, targets are lowered with
//     atomicMin (after a plain-load pre-filter); the first lowering of a vertex
//     in a round enqueues it exactly once (old == snapshot), so the next
//     frontier is duplicate-free without a bitmap pass.
#pragma once
#include "sg_ctl.cuh"

namespace sg {

constexpr int kTB = 256;        // threads per CTA of the traversal kernels
constexpr int kWarpsTB = kTB / 32;
constexpr uint32_t kLarge = 256;  // TWC CTA-bin cut (threads_per_cta, schedulers.py:159)
constexpr uint32_t kHugeSmem = 2048;  // huge prefixes staged in shared memory

struct PushArgs {
  const int64_t *off;
  const uint32_t *col;
  uint32_t nv;
  Ctl *ctl;
  uint32_t *q[2];
  uint32_t *largeq, *hugeq;
  int64_t *hpre, *hstart;
  unsigned long long *hval;
  const uint32_t *dying;  // src_mode 1: kcore dying list (count in ctl->ndying)
  int64_t threshold;      // huge threshold; INT64_MAX = twc (no huge bin)
  int src_mode;           // 0 frontier, 1 kcore dying list
  RoundStat *stats;
};

struct Src {
  const uint32_t *list;
  uint32_t n;
  bool dense;
};

__device__ __forceinline__ Src resolve_src(const PushArgs &a, const Ctl *c) {
  if (a.src_mode == 0) return {a.q[c->round & 1], c->dense ? a.nv : c->fsize, c->dense != 0};
  return {a.dying, c->ndying, false};
}

// ------------------------------------------------------------------ ops --
// bfs (OP_BFS): all frontier vertices of round r carry label r, so the source
// value is the round index; a visited bitmap is the relaxation test
// (label == inf <=> bit clear) and the atomicOr winner writes the label.
struct OpBfs {
  using L = uint32_t;
  uint32_t *lab, *vis;
  uint32_t r = 0;
  __device__ __forceinline__ void begin(uint32_t round) { r = round; }
  __device__ __forceinline__ L src_val(uint32_t) const { return r; }
  __device__ __forceinline__ bool relax(int64_t, uint32_t dst, L sv) const {
    uint32_t bit = 1u << (dst & 31u);
    uint32_t *wp = vis + (dst >> 5);
    if (*wp & bit) return false;
    if (atomicOr(wp, bit) & bit) return false;
    lab[dst] = sv + 1u;
    return true;
  }
};

// sssp / cc with 32-bit labels. KIND 0: cc (prop = value), 1: unit weight,
// 2: u32 weights.  Exact: integer sums below 2^32 equal the reference's
// float64 sums (the engine checks max_w * (V-1) < 2^32 - 1).
template <int KIND>
struct OpMin32 {
  using L = uint32_t;
  uint32_t *lab;
  const uint32_t *snap, *w;
  __device__ __forceinline__ void begin(uint32_t) {}
  __device__ __forceinline__ L src_val(uint32_t v) const { return snap[v]; }
  __device__ __forceinline__ bool relax(int64_t e, uint32_t dst, L sv) const {
    L prop = KIND == 0 ? sv : KIND == 1 ? sv + 1u : sv + __ldg(w + e);
    L cur = lab[dst];
    if (prop >= cur) return false;
    L old = atomicMin(lab + dst, prop);
    return prop < old && old == snap[dst];  // first lowering this round
  }
};

// sssp with float64 labels stored as their IEEE bits (labels >= 0, so
// unsigned order == numeric order): bit-exact to the reference for any
// non-negative int64 weights, including sums beyond 2^53.
struct OpMinF64 {
  using L = unsigned long long;
  unsigned long long *lab;
  const unsigned long long *snap;
  const int64_t *w;  // nullptr: unit weights
  __device__ __forceinline__ void begin(uint32_t) {}
  __device__ __forceinline__ L src_val(uint32_t v) const { return snap[v]; }
  __device__ __forceinline__ bool relax(int64_t e, uint32_t dst, L sv) const {
    double p = __dadd_rn(__longlong_as_double((long long)sv), w ? (double)w[e] : 1.0);
    L prop = (L)__double_as_longlong(p);
    L cur = lab[dst];
    if (prop >= cur) return false;
    L old = atomicMin(lab + dst, prop);
    return prop < old && old == snap[dst];
  }
};

// kcore dying-neighbour walk (apps.py:226-231): enqueue alive neighbours once.
struct OpMark {
  using L = uint32_t;
  const uint8_t *alive;
  uint32_t *mark;
  uint32_t stamp = 0;
  __device__ __forceinline__ void begin(uint32_t round) { stamp = round + 1; }
  __device__ __forceinline__ L src_val(uint32_t) const { return 0; }
  __device__ __forceinline__ bool relax(int64_t, uint32_t dst, L) const {
    if (!alive[dst]) return false;
    if (mark[dst] == stamp) return false;
    return atomicExch(mark + dst, stamp) != stamp;
  }
};

// --------------------------------------------------------------- kernels --
// inspection + TWC (small / medium by warp gathering); appends large / huge
template <class Op>
__global__ void __launch_bounds__(kTB) k_push_twc(PushArgs a, Op op) {
  __shared__ uint32_t sq[kWarpsTB][kWQ];
  __shared__ unsigned long long red[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  const Src src = resolve_src(a, ctl);
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  WarpQueue wq{sq[warp], 0, a.q[(round + 1) & 1], &ctl->nsize};
  unsigned long long my_edges = 0, my_large = 0;
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarpsTB;
  for (uint64_t c = (uint64_t)blockIdx.x * kWarpsTB + warp; c * 32 < src.n; c += nwarps) {
    uint64_t i = c * 32 + lane;
    uint32_t v = 0;
    int64_t s = 0, deg = 0;
    if (i < src.n) {
      v = src.dense ? (uint32_t)i : src.list[i];
      s = a.off[v];
      deg = a.off[v + 1] - s;
    }
    my_edges += (unsigned long long)deg;
    bool huge = deg >= a.threshold;
    bool large = !huge && deg >= (int64_t)kLarge;
    if (large) my_large += (unsigned long long)deg;
    warp_append(huge, v, a.hugeq, &ctl->nhuge);
    warp_append(large, v, a.largeq, &ctl->nlarge);
    uint32_t gd = (huge || large) ? 0u : (uint32_t)deg;
    typename Op::L sv = gd ? op.src_val(v) : typename Op::L(0);
    uint32_t incl = warp_incl_scan(gd);
    uint32_t total = __shfl_sync(kFull, incl, 31);
    uint32_t excl = incl - gd;
    for (uint32_t base = 0; base < total; base += 32) {
      uint32_t slot = base + lane;
      int o = warp_owner(incl, slot);
      int64_t so = shfl64(s, o);
      uint32_t eo = __shfl_sync(kFull, excl, o);
      typename Op::L svo = __shfl_sync(kFull, sv, o);
      bool act = false;
      uint32_t dst = 0;
      if (slot < total) {
        int64_t e = so + (slot - eo);
        dst = ld_stream(a.col + e);
        act = op.relax(e, dst, svo);
      }
      wq.push(act, dst);
    }
  }
  wq.flush();
  if (a.src_mode == 0) {
    unsigned long long bs = block_sum(my_edges, red);
    if (threadIdx.x == 0 && bs) atomicAdd(&ctl->edges, bs);
    bs = block_sum(my_large, red);
    if (threadIdx.x == 0 && bs) atomicAdd(&ctl->large_edges, bs);
  }
}

// TWC CTA bin: one CTA per vertex, dynamic fetch
template <class Op>
__global__ void __launch_bounds__(kTB) k_push_large(PushArgs a, Op op) {
  __shared__ uint32_t sq[kWarpsTB][kWQ];
  __shared__ uint32_t item;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  WarpQueue wq{sq[threadIdx.x >> 5], 0, a.q[(round + 1) & 1], &ctl->nsize};
  for (;;) {
    if (threadIdx.x == 0) item = atomicAdd(&ctl->large_head, 1u);
    __syncthreads();
    const uint32_t idx = item;
    __syncthreads();
    if (idx >= n) break;
    const uint32_t v = a.largeq[idx];
    const int64_t s = a.off[v], e = a.off[v + 1];
    const typename Op::L sv = op.src_val(v);
    for (int64_t b = s; b < e; b += kTB) {
      int64_t ei = b + threadIdx.x;
      bool act = false;
      uint32_t dst = 0;
      if (ei < e) {
        dst = ld_stream(a.col + ei);
        act = op.relax(ei, dst, sv);
      }
      wq.push(act, dst);
    }
  }
  wq.flush();
}

// PrefixWork for the huge list (worklist.py:68-93): inclusive int64 prefix of
// degrees in list order, plus each vertex's first edge and snapshot label.
template <class Op>
__global__ void __launch_bounds__(1024) k_huge_prefix(PushArgs a, Op op) {
  __shared__ long long red[32];
  __shared__ long long carry;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t n = ctl->nhuge;
  op.begin(ctl->round);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < n; b += 1024) {
    uint32_t i = b + threadIdx.x;
    long long d = 0;
    if (i < n) {
      uint32_t v = a.hugeq[i];
      a.hstart[i] = a.off[v];
      d = a.off[v + 1] - a.off[v];
      a.hval[i] = (unsigned long long)op.src_val(v);
    }
    long long x = warp_incl_scan(d);
    if (lane_id() == 31) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) red[threadIdx.x] = warp_incl_scan(red[threadIdx.x]);
    __syncthreads();
    long long wpre = (threadIdx.x >> 5) ? red[(threadIdx.x >> 5) - 1] : 0;
    if (i < n) a.hpre[i] = carry + wpre + x;
    __syncthreads();
    if (threadIdx.x == 1023) carry += wpre + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) ctl->huge_edges = (unsigned long long)carry;
}

// ALB huge-vertex kernel (Algorithm 2): every thread of every CTA
template <class Op, bool BLOCKED>
__global__ void __launch_bounds__(kTB) k_push_lb(PushArgs a, Op op) {
  __shared__ uint32_t sq[kWarpsTB][kWQ];
  __shared__ int64_t spre[kHugeSmem];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t nh = ctl->nhuge;
  if (!nh) return;
  const int64_t E = (int64_t)ctl->huge_edges;
  const uint32_t round = ctl->round;
  op.begin(round);
  const int64_t *pre = a.hpre;
  if (nh <= kHugeSmem) {
    for (uint32_t i = threadIdx.x; i < nh; i += kTB) spre[i] = a.hpre[i];
    __syncthreads();
    pre = spre;
  }
  WarpQueue wq{sq[threadIdx.x >> 5], 0, a.q[(round + 1) & 1], &ctl->nsize};
  const int64_t T = (int64_t)gridDim.x * kTB;
  const int64_t tid = (int64_t)blockIdx.x * kTB + threadIdx.x;
  const int64_t passes = (E + T - 1) / T;
  for (int64_t p = 0; p < passes; ++p) {
    // cyclic: g = p*T + tid (schedulers.py:191-194); blocked: g = tid*ceil(e/T) + p
    const int64_t g = BLOCKED ? tid * passes + p : p * T + tid;
    bool act = false;
    uint32_t dst = 0;
    if (g < E) {
      uint32_t o = owner_search(pre, nh, g);
      int64_t e = a.hstart[o] + (g - (o ? pre[o - 1] : 0));
      dst = ld_stream(a.col + e);
      act = op.relax(e, dst, (typename Op::L)a.hval[o]);
    }
    wq.push(act, dst);
  }
  wq.flush();
}

}  // namespace sg
