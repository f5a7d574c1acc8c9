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
//   * CTA bin: one CTA per vertex (static round robin, no barriers);
//   * huge bin: a single-CTA scan builds the int64 prefix + snapshot labels, the
//     LB kernel stages the prefix in shared memory and every thread of every CTA
//     walks g cyclically: consecutive lanes read consecutive adjacency entries;
//   * every lane relaxes kU edges per step, in phases (adjacency loads, label
//     loads, atomics), so kU independent random accesses are in flight;
//   * BSP without a commit pass: labels are parity pairs {L0, L1}; round r reads
//     half r&1 (a snapshot nobody writes during the round) and lowers half
//     (r+1)&1.  Frontier vertices re-sync their next half with one red.min; the
//     first atomicMin that takes a vertex below its snapshot (old >= snapshot)
//     enqueues it, so the next frontier is exact and duplicate-free.
#pragma once
#include "sg_ctl.cuh"

namespace sg {

constexpr int kTB = 256;        // threads per CTA of the traversal kernels
constexpr int kWarpsTB = kTB / 32;
#ifndef SG_KU
#define SG_KU 4
#endif
constexpr int kU = SG_KU;       // edges per lane per step (memory-level parallelism)
constexpr uint32_t kLarge = 256;  // TWC CTA-bin cut (threads_per_cta, schedulers.py:159)
constexpr uint32_t kHugeSmem = 1024;  // huge-vertex prefix/start/label staged in shared memory
static_assert(kHugeSmem >= 256, "k_bm_lb reuses spre for the 256-entry Coarse sample");
constexpr uint32_t kChunkGrab = 4;    // TWC chunks (32 items each) per dynamic fetch
constexpr int kBatch = 32;            // CTA-bin vertices per block-level gather batch

struct PushArgs {
  const int64_t *off;
  const uint32_t *col;
  uint32_t nv;
  Ctl *ctl;
  uint32_t *q[2];
  uint32_t *largeq, *hugeq;
  int64_t *hpre, *hstart;
  unsigned long long *hval;
  unsigned long long *largesv;  // snapshot labels of the CTA-bin queue (Op::kCarry)
  const uint32_t *dying;  // src_mode 1: kcore dying list (count in ctl->ndying)
  int64_t threshold;      // huge threshold; INT64_MAX = twc (no huge bin)
  int src_mode;           // 0 frontier, 1 kcore dying list
  RoundStat *stats;
  int no_enqueue;         // partitioned runs: frontiers come from the label exchange
  int sched;              // 0 alb / twc, 1 lb, 2 vertex, 3 edge (round-log launch accounting)
  uint32_t dense_lo, dense_n;  // a dense frontier is [dense_lo, dense_lo + dense_n)
  // vertices >= zlo have no out-edges in this view (relabeled store: they are
  // numbered last); the compaction counts them instead of queueing them
  uint32_t zlo = 0xffffffffu;
  int prefix_in_large = 0;  // the CTA-bin kernel's CTA 0 builds the huge prefix (no k_huge_prefix)
  // SG_FLAG_CTA_COUNTS: edges processed per CTA per round ([round][cta_g]), the
  // hardware analogue of the reference's modeled per-CTA counters
  unsigned long long *cta_edges;
  uint32_t cta_g, cta_rounds;
};

// counters are kept per SM (the slot a CTA ran on): the persistent grids of
// the round's kernels differ in size, SMs are the fixed resource they share
__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
template <class Args>
__device__ __forceinline__ void cta_flush(const Args &a, unsigned long long n, uint32_t round) {
  if (a.cta_edges && n && round < a.cta_rounds)
    atomicAdd(a.cta_edges + (size_t)round * a.cta_g + (sm_id() % a.cta_g), n);
}
template <int N>
__device__ __forceinline__ unsigned count_ok(const bool (&ok)[N]) {
  unsigned c = 0;
#pragma unroll
  for (int u = 0; u < N; ++u) c += ok[u];
  return c;
}

__device__ __forceinline__ uint32_t *next_queue(const PushArgs &a, uint32_t round) {
  return a.no_enqueue ? nullptr : ((round & 1) ? a.q[0] : a.q[1]);
}

struct Src {
  const uint32_t *list;
  uint32_t n;
  bool dense;
  uint32_t lo;
  __device__ __forceinline__ uint32_t at(uint64_t i) const {
    return dense ? lo + (uint32_t)i : list[i];
  }
};

__device__ __forceinline__ Src resolve_src(const PushArgs &a, const Ctl *c) {
  if (a.src_mode == 0)
    return {((c->round & 1) ? a.q[1] : a.q[0]), c->dense ? a.dense_n : c->fsize, c->dense != 0,
            a.dense_lo};
  return {a.dying, c->ndying, false, 0};
}

// ------------------------------------------------------------------ ops --
// Every op relaxes kU edges at once: relax(e, valid, sv, dst, act).
// bfs (OP_BFS): frontier vertices of round r carry label r; a visited bitmap
// is the relaxation test (label == inf <=> bit clear); the atomicOr winner
// writes the label.
struct OpBfs {
  using L = uint32_t;
  uint32_t *lab, *vis;
  uint32_t r = 0;
  __device__ __forceinline__ void begin(uint32_t round) { r = round; }
  static constexpr bool kCarry = false;
  __device__ __forceinline__ L src_val(uint64_t, uint32_t) const { return r; }
  __device__ __forceinline__ void sync_src(uint32_t, L) const {}
  __device__ __forceinline__ void relax(const PushArgs &a, const int64_t (&e)[kU],
                                        const bool (&ok)[kU], const L (&sv)[kU],
                                        uint32_t (&dst)[kU], bool (&act)[kU]) const {
    uint32_t word[kU], old[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u) word[u] = ok[u] ? vis[dst[u] >> 5] : ~0u;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint32_t bit = 1u << (dst[u] & 31u);
      old[u] = (word[u] & bit) ? bit : atomicOr(vis + (dst[u] >> 5), bit);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      act[u] = ok[u] && !(old[u] & (1u << (dst[u] & 31u)));
      if (act[u]) lab[dst[u]] = sv[u] + 1u;
    }
  }
};

// sssp / cc on parity-paired labels.  KIND 0: cc (prop = value), 1: unit
// weight, 2: u32 weights, 3: float64 labels (bits) with int64 weights.
// 32-bit kinds are exact: integer sums below 2^32 equal the reference's
// float64 sums (the engine checks max_w * (V-1) < 2^32 - 1); kind 3 performs
// the reference's float64 additions (labels >= 0, so unsigned bit order ==
// numeric order and atomicMin on the bits is a float min).
template <int KIND>
struct OpPair {
  using L = typename std::conditional<KIND == 3, unsigned long long, uint32_t>::type;
  L *lab;  // lab[2v + h]
  const uint32_t *w32;
  const int64_t *w64;  // KIND 3 (nullptr: unit weights)
  uint32_t ch = 0, nh = 1;  // current (snapshot) / next half
  __device__ __forceinline__ void begin(uint32_t round) { ch = round & 1u, nh = ch ^ 1u; }
  static constexpr bool kCarry = false;
  __device__ __forceinline__ L src_val(uint64_t, uint32_t v) const {
    return lab[2 * (size_t)v + ch];
  }
  // a frontier vertex changed last round: its next half still holds the older value
  __device__ __forceinline__ void sync_src(uint32_t v, L sv) const {
    atomicMin(lab + 2 * (size_t)v + nh, sv);
  }
  __device__ __forceinline__ L prop(int64_t e, L sv) const {
    if (KIND == 0) return sv;
    if (KIND == 1) return sv + 1u;
    if (KIND == 2) return sv + ld_stream(w32 + e);
    double p = __dadd_rn(__longlong_as_double((long long)sv), w64 ? (double)ld_stream(w64 + e) : 1.0);
    return (L)__double_as_longlong(p);
  }
  __device__ __forceinline__ void relax(const PushArgs &a, const int64_t (&e)[kU],
                                        const bool (&ok)[kU], const L (&sv)[kU],
                                        uint32_t (&dst)[kU], bool (&act)[kU]) const {
    L p[kU], cur[kU], nxt[kU], old[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      p[u] = ok[u] ? prop(e[u], sv[u]) : L(0);
      if (KIND == 3) {
        ulonglong2 pr = ok[u] ? reinterpret_cast<const ulonglong2 *>(lab)[dst[u]]
                              : make_ulonglong2(0, 0);
        cur[u] = ch ? pr.y : pr.x;
        nxt[u] = ch ? pr.x : pr.y;
      } else {
        uint2 pr = ok[u] ? reinterpret_cast<const uint2 *>(lab)[dst[u]] : make_uint2(0, 0);
        cur[u] = ch ? pr.y : pr.x;
        nxt[u] = ch ? pr.x : pr.y;
      }
    }
    bool t[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {  // issue all atomics before consuming any result
      t[u] = ok[u] && p[u] < cur[u] && p[u] < nxt[u];
      old[u] = t[u] ? atomicMin(lab + 2 * (size_t)dst[u] + nh, p[u]) : L(0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) act[u] = t[u] && old[u] >= cur[u];  // first drop below snapshot
  }
};

// kcore dying-neighbour walk (apps.py:226-231): enqueue alive neighbours once.
struct OpMark {
  using L = uint32_t;
  const uint8_t *alive;
  uint32_t *mark;
  uint32_t stamp = 0;
  __device__ __forceinline__ void begin(uint32_t round) { stamp = round + 1; }
  static constexpr bool kCarry = false;
  __device__ __forceinline__ L src_val(uint64_t, uint32_t) const { return 0; }
  __device__ __forceinline__ void sync_src(uint32_t, L) const {}
  __device__ __forceinline__ void relax(const PushArgs &a, const int64_t (&e)[kU],
                                        const bool (&ok)[kU], const L (&)[kU],
                                        uint32_t (&dst)[kU], bool (&act)[kU]) const {
    bool t[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u) t[u] = ok[u] && alive[dst[u]] && mark[dst[u]] != stamp;
    uint32_t old[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) old[u] = t[u] ? atomicExch(mark + dst[u], stamp) : stamp;
#pragma unroll
    for (int u = 0; u < kU; ++u) act[u] = old[u] != stamp;
  }
};

// --------------------------------------------------------------- kernels --
// inspection + TWC (small / medium by warp gathering); appends large / huge
template <class Op>
__global__ void __launch_bounds__(kTB) k_push_twc(PushArgs a, Op op) {
  using L = typename Op::L;
  __shared__ uint32_t sq[kWarpsTB][kWQ];
  __shared__ unsigned long long red[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  const Src src = resolve_src(a, ctl);
  const bool sync = a.src_mode == 0 && round > 0;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  WarpQueue wq{sq[warp], 0, next_queue(a, round), &ctl->nsize};
  unsigned long long my_edges = 0, my_large = 0;
  // dynamic fetch: a warp grabs kChunkGrab chunks of 32 frontier items at a time
  const uint32_t nchunks = (src.n + 31) / 32;
  // a frontier of at most one chunk per warp: warp w takes chunk w and no
  // warp touches the shared counter (a small round's chunks then run in
  // parallel instead of kChunkGrab-deep on a few warps); otherwise dynamic
  // grabs of kChunkGrab chunks
  const bool small = nchunks <= grid_warps();
  uint32_t c = 0, c_end = 0;
  if (small) {
    c = global_warp();
    c_end = c < nchunks ? c + 1 : c;
  }
  for (;;) {
    if (c == c_end) {
      if (small) break;
      uint32_t g = 0;
      if (lane == 0) g = atomicAdd(&ctl->chunk_head, 1u);
      g = __shfl_sync(kFull, g, 0);
      c = g * kChunkGrab;
      if (c >= nchunks) break;
      c_end = min(c + kChunkGrab, nchunks);
    }
    uint64_t i = (uint64_t)c * 32 + lane;
    ++c;
    uint32_t v = 0;
    int64_t s = 0, deg = 0;
    L sv = 0;
    if (i < src.n) {
      v = src.at(i);
      s = a.off[v];
      deg = a.off[v + 1] - s;
      sv = op.src_val(i, v);
      if (sync) op.sync_src(v, sv);
    }
    my_edges += (unsigned long long)deg;
    const bool huge = deg >= a.threshold;
    const bool large = !huge && deg >= (int64_t)kLarge;
    if (large) my_large += (unsigned long long)deg;
    const uint32_t hslot = warp_append(huge, v, a.hugeq, &ctl->nhuge);
    const uint32_t lslot = warp_append(large, v, a.largeq, &ctl->nlarge);
    if (Op::kCarry) {
      if (huge) a.hval[hslot] = (unsigned long long)sv;
      if (large) a.largesv[lslot] = (unsigned long long)sv;
    }
    const uint32_t gd = (huge || large) ? 0u : (uint32_t)deg;
    const uint32_t incl = warp_incl_scan(gd);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - gd;
    for (uint32_t base = 0; base < total; base += 32 * kU) {
      int64_t e[kU];
      bool ok[kU];
      L svo[kU];
      uint32_t dst[kU];
      bool act[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t slot = base + u * 32 + lane;
        const int o = warp_owner(incl, slot);
        const int64_t so = shfl64(s, o);
        const uint32_t eo = __shfl_sync(kFull, excl, o);
        svo[u] = __shfl_sync(kFull, sv, o);
        ok[u] = slot < total;
        e[u] = so + (int64_t)(slot - eo);
      }
      op.relax(a, e, ok, svo, dst, act);
#pragma unroll
      for (int u = 0; u < kU; ++u) wq.push(act[u], dst[u]);
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

// TWC CTA bin: one CTA per vertex, static round robin (no barriers)
template <class Op>
__global__ void __launch_bounds__(kTB) k_push_large(PushArgs a, Op op) {
  using L = typename Op::L;
  __shared__ uint32_t sq[kWarpsTB][kWQ];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  WarpQueue wq{sq[threadIdx.x >> 5], 0, next_queue(a, round), &ctl->nsize};
  // Block-level gather over batches of kBatch CTA-bin vertices: the batch's
  // edges are numbered through a shared-memory prefix and all 256 x kU slots
  // of each step are filled, whatever the individual degrees are.
  __shared__ int64_t bstart[kBatch];
  __shared__ long long bexcl[kBatch + 1];
  __shared__ L bsv[kBatch];
  __shared__ uint32_t bhead;
  // batch b takes queue entries b, b+NB, b+2NB, ... so that batches mix the
  // (degree-correlated) queue order and carry similar edge totals
  const uint32_t nb = (n + kBatch - 1) / kBatch;
  bool first_grab = true;
  for (;;) {
    if (threadIdx.x == 0) bhead = cta_grab(&ctl->large_head, first_grab);
    __syncthreads();
    const uint32_t bidx = bhead;
    if (bidx >= nb) break;
    if (threadIdx.x < 32) {
      const uint32_t i = bidx + threadIdx.x * nb;
      long long d = 0;
      if (threadIdx.x < kBatch && i < n) {
        const uint32_t v = a.largeq[i];
        const int64_t s = a.off[v];
        d = a.off[v + 1] - s;
        bstart[threadIdx.x] = s;
        bsv[threadIdx.x] = Op::kCarry ? (L)a.largesv[i] : op.src_val(i, v);
      }
      const long long incl = warp_incl_scan(d);
      if (threadIdx.x < kBatch) bexcl[threadIdx.x + 1] = incl;
      if (threadIdx.x == 0) bexcl[0] = 0;
    }
    __syncthreads();
    const long long total = bexcl[kBatch];
    for (long long b = 0; b < total; b += kTB * kU) {
      int64_t e[kU];
      bool ok[kU];
      L svs[kU];
      uint32_t dst[kU];
      bool act[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const long long slot = b + u * kTB + threadIdx.x;
        ok[u] = slot < total;
        uint32_t lo = 0;  // owner: last o with bexcl[o] <= slot (branchless, kBatch == 32)
#pragma unroll
        for (uint32_t step = kBatch / 2; step; step >>= 1)
          lo = bexcl[lo + step] <= slot ? lo + step : lo;
        e[u] = bstart[lo] + (slot - bexcl[lo]);
        svs[u] = bsv[lo];
      }
      op.relax(a, e, ok, svs, dst, act);
#pragma unroll
      for (int u = 0; u < kU; ++u) wq.push(act[u], dst[u]);
    }
    __syncthreads();
  }
  wq.flush();
}

// PrefixWork for the huge list (worklist.py:68-93): inclusive int64 prefix of
// degrees in list order, plus each vertex's first edge and snapshot label.
template <class Op>
__global__ void __launch_bounds__(1024) k_huge_prefix(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
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
      if (!Op::kCarry) a.hval[i] = (unsigned long long)op.src_val(i, v);
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
  using L = typename Op::L;
  __shared__ uint32_t sq[kWarpsTB][kWQ];
  __shared__ int64_t spre[kHugeSmem], sstart[kHugeSmem];
  __shared__ unsigned long long sval[kHugeSmem];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t nh = ctl->nhuge;
  if (!nh) return;
  const int64_t E = (int64_t)ctl->huge_edges;
  const uint32_t round = ctl->round;
  op.begin(round);
  const bool staged = nh <= kHugeSmem;
  if (staged) {
    for (uint32_t i = threadIdx.x; i < nh; i += kTB)
      spre[i] = a.hpre[i], sstart[i] = a.hstart[i], sval[i] = a.hval[i];
    __syncthreads();
  }
  WarpQueue wq{sq[threadIdx.x >> 5], 0, next_queue(a, round), &ctl->nsize};
  const int64_t T = (int64_t)gridDim.x * kTB;
  const int64_t tid = (int64_t)blockIdx.x * kTB + threadIdx.x;
  const int64_t passes = (E + T - 1) / T;
  for (int64_t p0 = 0; p0 < passes; p0 += kU) {
    int64_t e[kU];
    bool ok[kU];
    L sv[kU];
    uint32_t dst[kU];
    bool act[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      // cyclic: g = p*T + tid (schedulers.py:191-194); blocked: g = tid*ceil(e/T) + p
      const int64_t p = p0 + u;
      const int64_t g = BLOCKED ? tid * passes + p : p * T + tid;
      ok[u] = p < passes && g < E;
      const int64_t gg = ok[u] ? g : 0;
      if (staged) {  // shared-memory bisection (LDS), find_owner (worklist.py:96-119)
        const uint32_t o = owner_search(spre, nh, gg);
        e[u] = sstart[o] + (gg - (o ? spre[o - 1] : 0));
        sv[u] = (L)sval[o];
      } else {
        const uint32_t o = owner_search(a.hpre, nh, gg);
        e[u] = a.hstart[o] + (gg - (o ? a.hpre[o - 1] : 0));
        sv[u] = (L)a.hval[o];
      }
    }
    op.relax(a, e, ok, sv, dst, act);
#pragma unroll
    for (int u = 0; u < kU; ++u) wq.push(act[u], dst[u]);
  }
  wq.flush();
}

}  // namespace sg
