// sg_bm.cuh — single-device ALB push round with a bitmap next-frontier.
//
// Same bins and operator as sg_push.cuh (inspection fused into TWC, CTA bin,
// huge-vertex LB kernel; schedulers.py:252-298, _kernels_py.py:69-85), but
// the relaxation never waits for an atomic result:
//
//   candidate  : p < lab[dst]  (any read during the round is <= the round-start
//                snapshot, because labels only decrease; an L1-stale value is
//                only ever too high, so it can add candidates, never drop one)
//   update     : red.min(lab[dst], p); red.or(next_bitmap[dst / 32], bit)
//
// A candidate's label ends the round <= p < snapshot, so it changed; a vertex
// that changed had a lowering thread whose earlier read was > p, so it was a
// candidate.  Hence the bitmap is exactly {v : merged[v] < values[v]}, the
// reference's next frontier (apps.py:71-74), and k_bm_compact turns it into an
// ascending-within-warp id list plus each vertex's snapshot label.
//
// Why: a scattered 4-byte access costs one L1TEX wavefront per lane; the chip
// sustains ~275 G of them per second (measured, scripts/micro/gather.cu).
// Atomics with return values add a full round trip per step on top, so the
// hot kernels issue only fire-and-forget reductions and keep kV independent
// gathers in flight per lane.
#pragma once
#include "sg_push.cuh"

namespace sg {

#ifndef SG_BKV
#define SG_BKV 6
#endif
constexpr int kV = SG_BKV;
#ifndef SG_LB_STEPS
#define SG_LB_STEPS 4
#endif
constexpr int kLBSteps = SG_LB_STEPS;  // relax steps of 32 x kV edges per LB chunk (per bisection)  // edges per lane per step in the bitmap-frontier kernels
static_assert(kV * 32 <= (int)kLarge, "k_bm_large: a warp step must span <= 2 CTA-bin vertices");

// bfs: frontier vertices of round r carry label r.  vis = visited bitmap
// (red.or during the round); prev = vis as of the round start, so the next
// frontier is vis & ~prev; the compaction writes label r + 1.
struct BmBfs {
  using L = uint32_t;
  static constexpr bool kCarry = true;
  uint32_t *lab, *vis, *prev;
  uint32_t r = 0;
  __device__ __forceinline__ void begin(uint32_t round) { r = round; }
  __device__ __forceinline__ L src_val(uint64_t, uint32_t) const { return r; }
  __device__ __forceinline__ void relax(const PushArgs &a, const int64_t (&e)[kV],
                                        const bool (&ok)[kV], const L (&)[kV]) const {
    uint32_t dst[kV], w[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
#pragma unroll
    for (int u = 0; u < kV; ++u) w[u] = ok[u] ? vis[dst[u] >> 5] : ~0u;
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const uint32_t bit = 1u << (dst[u] & 31u);
      if (!(w[u] & bit)) atomicOr(vis + (dst[u] >> 5), bit);  // RED.OR (result unused)
    }
  }
  using W = uint32_t;
  template <int N>
  __device__ __forceinline__ void fetch(const PushArgs &a, const int64_t (&e)[N],
                                        const bool (&ok)[N], uint32_t (&dst)[N],
                                        W (&)[N]) const {
#pragma unroll
    for (int u = 0; u < N; ++u) dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
  }
  template <int N>
  __device__ __forceinline__ void apply(const uint32_t (&dst)[N], const W (&)[N], const L (&)[N],
                                        const bool (&ok)[N]) const {
    uint32_t w[N];
#pragma unroll
    for (int u = 0; u < N; ++u) w[u] = ok[u] ? vis[dst[u] >> 5] : ~0u;
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const uint32_t bit = 1u << (dst[u] & 31u);
      if (!(w[u] & bit)) atomicOr(vis + (dst[u] >> 5), bit);
    }
  }
  // new bits of word wi (and advance prev)
  __device__ __forceinline__ uint32_t take(uint32_t wi) const {
    const uint32_t x = vis[wi], n = x & ~prev[wi];
    if (n) prev[wi] = x;
    return n;
  }
  // compaction: per emitted vertex, a load (none here) and the stores
  using E = uint32_t;
  __device__ __forceinline__ E emit_load(uint32_t) const { return 0u; }
  __device__ __forceinline__ void emit_store(uint32_t, uint32_t v, E) const { lab[v] = r + 1; }
  __device__ __forceinline__ void emit_zero(uint32_t v) const { lab[v] = r + 1; }
};

// sssp / cc (KIND as OpPair: 0 cc, 1 unit weight, 2 u32 weights, 3 float64 bits)
template <int KIND>
struct BmMin {
  using L = typename std::conditional<KIND == 3, unsigned long long, uint32_t>::type;
  static constexpr bool kCarry = true;
  L *lab;
  const uint32_t *w32;
  const int64_t *w64;  // KIND 3 (nullptr: unit weights)
  L *snap;             // snapshot label per frontier slot (written by k_bm_compact)
  uint32_t *nb;        // next-frontier bitmap
  __device__ __forceinline__ void begin(uint32_t) {}
  __device__ __forceinline__ L src_val(uint64_t i, uint32_t) const { return snap[i]; }
  __device__ __forceinline__ L prop(int64_t e, L sv) const {
    if (KIND == 0) return sv;
    if (KIND == 1) return sv + 1u;
    if (KIND == 2) return sv + ld_stream(w32 + e);
    double p = __dadd_rn(__longlong_as_double((long long)sv), w64 ? (double)ld_stream(w64 + e) : 1.0);
    return (L)__double_as_longlong(p);
  }
  __device__ __forceinline__ void relax(const PushArgs &a, const int64_t (&e)[kV],
                                        const bool (&ok)[kV], const L (&sv)[kV]) const {
    uint32_t dst[kV];
    L p[kV], cur[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
#pragma unroll
    for (int u = 0; u < kV; ++u) p[u] = ok[u] ? prop(e[u], sv[u]) : L(0);
#pragma unroll
    for (int u = 0; u < kV; ++u) cur[u] = ok[u] ? lab[dst[u]] : L(0);
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      if (p[u] < cur[u]) {  // ok[u] implied: cur = 0 otherwise
        atomicMin(lab + dst[u], p[u]);                      // RED.MIN
        atomicOr(nb + (dst[u] >> 5), 1u << (dst[u] & 31u));  // RED.OR
      }
    }
  }
  // split relax for software-pipelined loops: fetch (adjacency + weight
  // loads) of step k+1 is issued before apply (label gathers + reductions)
  // of step k
  using W = typename std::conditional<KIND == 3, int64_t, uint32_t>::type;
  template <int N>
  __device__ __forceinline__ void fetch(const PushArgs &a, const int64_t (&e)[N],
                                        const bool (&ok)[N], uint32_t (&dst)[N],
                                        W (&w)[N]) const {
#pragma unroll
    for (int u = 0; u < N; ++u) {
      dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
      if (KIND == 2) w[u] = ok[u] ? ld_stream(w32 + e[u]) : 0u;
      if (KIND == 3) w[u] = (ok[u] && w64) ? ld_stream(w64 + e[u]) : (W)1;
    }
  }
  template <int N>
  __device__ __forceinline__ void apply(const uint32_t (&dst)[N], const W (&w)[N],
                                        const L (&sv)[N], const bool (&ok)[N]) const {
    L p[N], cur[N];
#pragma unroll
    for (int u = 0; u < N; ++u) {
      if (KIND == 0) p[u] = sv[u];
      else if (KIND == 1) p[u] = sv[u] + 1u;
      else if (KIND == 2) p[u] = sv[u] + (uint32_t)w[u];
      else p[u] = (L)__double_as_longlong(
               __dadd_rn(__longlong_as_double((long long)sv[u]), (double)w[u]));
      cur[u] = ok[u] ? lab[dst[u]] : L(0);
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
      if (ok[u] && p[u] < cur[u]) {
        atomicMin(lab + dst[u], p[u]);
        atomicOr(nb + (dst[u] >> 5), 1u << (dst[u] & 31u));
      }
    }
  }
  __device__ __forceinline__ uint32_t take(uint32_t wi) const {
    const uint32_t x = nb[wi];
    if (x) nb[wi] = 0u;
    return x;
  }
  using E = L;
  __device__ __forceinline__ E emit_load(uint32_t v) const { return lab[v]; }
  __device__ __forceinline__ void emit_store(uint32_t slot, uint32_t, E x) const { snap[slot] = x; }
  __device__ __forceinline__ void emit_zero(uint32_t) const {}
};

// ---------------------------------------------------------------- kernels --
// inspection + TWC small/medium (warp gather); huge / CTA-bin vertices are
// queued with their snapshot label
// resident CTAs per SM the TWC kernel is compiled for (the register cap that
// keeps each operator at the occupancy it was measured best with: bfs 40
// registers / 6 CTAs, 4-byte labels 48 / 5, 8-byte labels 64 / 4)
template <class Op>
constexpr int twc_min_blocks() {
  return std::is_same<Op, BmBfs>::value ? 6 : sizeof(typename Op::L) == 8 ? 4 : 5;
}

template <class Op>
__global__ void __launch_bounds__(kTB, twc_min_blocks<Op>()) k_bm_twc(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
  using L = typename Op::L;
  __shared__ unsigned long long red[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  unsigned long long my_proc = 0;
  const Src src = resolve_src(a, ctl);
  const uint32_t lane = lane_id();
  unsigned long long my_edges = 0, my_large = 0;
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
    const uint64_t i = (uint64_t)c * 32 + lane;
    ++c;
    uint32_t v = 0;
    int64_t s = 0, deg = 0;
    L sv = 0;
    if (i < src.n) {
      v = src.at(i);
      s = a.off[v];
      deg = a.off[v + 1] - s;
      sv = op.src_val(i, v);
    }
    my_edges += (unsigned long long)deg;
    const bool huge = deg >= a.threshold;
    const bool large = !huge && deg >= (int64_t)kLarge;
    if (large) my_large += (unsigned long long)deg;
    const uint32_t hslot = warp_append(huge, v, a.hugeq, &ctl->nhuge);
    const uint32_t lslot = warp_append(large, v, a.largeq, &ctl->nlarge);
    if (huge) a.hval[hslot] = (unsigned long long)sv;
    if (large) a.largesv[lslot] = (unsigned long long)sv;
    const uint32_t gd = (huge || large) ? 0u : (uint32_t)deg;
    const uint32_t incl = warp_incl_scan(gd);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - gd;
    for (uint32_t base = 0; base < total; base += 32 * kV) {
      int64_t e[kV];
      bool ok[kV];
      L svo[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const uint32_t slot = base + u * 32 + lane;
        const int o = warp_owner(incl, slot);
        const int64_t so = shfl64(s, o);
        const uint32_t eo = __shfl_sync(kFull, excl, o);
        svo[u] = __shfl_sync(kFull, sv, o);
        ok[u] = slot < total;
        e[u] = so + (int64_t)(slot - eo);
      }
      if (a.cta_edges) my_proc += count_ok(ok);
      op.relax(a, e, ok, svo);
    }
  }
  unsigned long long bs = block_sum(my_edges, red);
  if (threadIdx.x == 0 && bs) atomicAdd(&ctl->edges, bs);
  bs = block_sum(my_large, red);
  if (threadIdx.x == 0 && bs) atomicAdd(&ctl->large_edges, bs);
  cta_flush(a, my_proc, ctl->round);
}

// ALB's PrefixWork (worklist.py:68-93) of the huge vertices the inspection
// queued, by one CTA of any size: hstart, inclusive hpre, ctl->huge_edges.
// The CTA-bin kernel's CTA 0 runs it before its batches (a.prefix_in_large),
// which saves the round a kernel node; the LB kernel runs after the CTA bin.
template <class Op>
__device__ void huge_prefix_cta(const PushArgs &a, Op &op) {
  __shared__ long long red[32];
  __shared__ long long carry;
  Ctl *ctl = a.ctl;
  const uint32_t n = ctl->nhuge;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < n; b += blockDim.x) {
    const uint32_t i = b + threadIdx.x;
    long long d = 0;
    if (i < n) {
      const uint32_t v = a.hugeq[i];
      const int64_t s0 = a.off[v];
      a.hstart[i] = s0;
      d = a.off[v + 1] - s0;
      if (!Op::kCarry) a.hval[i] = (unsigned long long)op.src_val(i, v);
    }
    const long long x = warp_incl_scan(d);
    if (lane_id() == 31) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      const long long y = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
      red[threadIdx.x] = warp_incl_scan(y);
    }
    __syncthreads();
    const long long wpre = (threadIdx.x >> 5) ? red[(threadIdx.x >> 5) - 1] : 0;
    if (i < n) a.hpre[i] = carry + wpre + x;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += wpre + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) ctl->huge_edges = (unsigned long long)carry;
}

// TWC CTA bin: block-level gather over batches of kBatch queued vertices
template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_large(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
  using L = typename Op::L;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  if (a.prefix_in_large && blockIdx.x == 0 && ctl->nhuge) huge_prefix_cta(a, op);
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  __shared__ int64_t bstart[kBatch];
  __shared__ long long bexcl[kBatch + 1];
  __shared__ L bsv[kBatch];
  __shared__ uint32_t bhead;
  const uint32_t nb = (n + kBatch - 1) / kBatch;
  bool first_grab = true;
  for (;;) {
    if (threadIdx.x == 0) bhead = cta_grab(&ctl->large_head, first_grab);
    __syncthreads();
    const uint32_t bidx = bhead;
    if (bidx >= nb) break;
    if (threadIdx.x < 32) {
      const uint32_t i = bidx + threadIdx.x * nb;  // degree-mixed batch
      long long d = 0;
      if (threadIdx.x < kBatch && i < n) {
        const uint32_t v = a.largeq[i];
        const int64_t s = a.off[v];
        d = a.off[v + 1] - s;
        bstart[threadIdx.x] = s;
        bsv[threadIdx.x] = (L)a.largesv[i];
      }
      const long long incl = warp_incl_scan(d);
      if (threadIdx.x < kBatch) bexcl[threadIdx.x + 1] = incl;
      if (threadIdx.x == 0) bexcl[0] = 0;
    }
    __syncthreads();
    const long long total = bexcl[kBatch];
    // each warp takes 32*kV consecutive slots per step; every CTA-bin vertex
    // owns >= kLarge >= 32*kV slots, so they span at most two owners: one
    // warp-uniform bisection (shared-memory broadcast) per step, then a
    // compare per slot
    for (long long b = 0; b < total; b += kTB * kV) {
      const long long wbase = b + (long long)(threadIdx.x >> 5) * (32 * kV);
      uint32_t lo = 0;  // last o with bexcl[o] <= wbase (kBatch == 32)
#pragma unroll
      for (uint32_t step = kBatch / 2; step; step >>= 1)
        lo = bexcl[lo + step] <= wbase ? lo + step : lo;
      const long long x0 = bexcl[lo], x1 = bexcl[lo + 1];
      const int64_t s0 = bstart[lo], s1 = lo + 1 < kBatch ? bstart[lo + 1] : 0;
      const L v0 = bsv[lo], v1 = lo + 1 < kBatch ? bsv[lo + 1] : L(0);
      int64_t e[kV];
      bool ok[kV];
      L svs[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const long long slot = wbase + u * 32 + (threadIdx.x & 31u);
        ok[u] = slot < total;
        const bool second = slot >= x1;
        e[u] = second ? s1 + (slot - x1) : s0 + (slot - x0);
        svs[u] = second ? v1 : v0;
      }
      if (a.cta_edges) my_proc += count_ok(ok);
      op.relax(a, e, ok, svs);
    }
    __syncthreads();
  }
  cta_flush(a, my_proc, ctl->round);
}

#ifndef SG_PIPE_V
#define SG_PIPE_V 4
#endif
constexpr int kPV = SG_PIPE_V;  // edges per lane per step of the pipelined CTA-bin loop

// CTA bin, software-pipelined: the adjacency (+ weight) loads of step k+1 are
// in flight while step k's label gathers and reductions issue
template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_large_pipe(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
  using L = typename Op::L;
  using W = typename Op::W;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  if (a.prefix_in_large && blockIdx.x == 0 && ctl->nhuge) huge_prefix_cta(a, op);
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  __shared__ int64_t bstart[kBatch];
  __shared__ long long bexcl[kBatch + 1];
  __shared__ L bsv[kBatch];
  __shared__ uint32_t bhead;
  const uint32_t nb = (n + kBatch - 1) / kBatch;
  const long long wstep = 32 * kPV, step = (long long)kTB * kPV;
  const long long woff = (long long)(threadIdx.x >> 5) * wstep;
  const uint32_t lane = threadIdx.x & 31u;
  bool first_grab = true;
  for (;;) {
    if (threadIdx.x == 0) bhead = cta_grab(&ctl->large_head, first_grab);
    __syncthreads();
    const uint32_t bidx = bhead;
    if (bidx >= nb) break;
    if (threadIdx.x < 32) {
      const uint32_t i = bidx + threadIdx.x * nb;  // degree-mixed batch
      long long d = 0;
      if (threadIdx.x < kBatch && i < n) {
        const uint32_t v = a.largeq[i];
        const int64_t s = a.off[v];
        d = a.off[v + 1] - s;
        bstart[threadIdx.x] = s;
        bsv[threadIdx.x] = (L)a.largesv[i];
      }
      const long long incl = warp_incl_scan(d);
      if (threadIdx.x < kBatch) bexcl[threadIdx.x + 1] = incl;
      if (threadIdx.x == 0) bexcl[0] = 0;
    }
    __syncthreads();
    const long long total = bexcl[kBatch];
    auto slots = [&](long long b, int64_t (&e)[kPV], bool (&ok)[kPV], L (&sv)[kPV]) {
      const long long wbase = b + woff;
      uint32_t lo = 0;
#pragma unroll
      for (uint32_t st = kBatch / 2; st; st >>= 1) lo = bexcl[lo + st] <= wbase ? lo + st : lo;
      const long long x0 = bexcl[lo], x1 = bexcl[lo + 1];
      const int64_t s0 = bstart[lo], s1 = lo + 1 < kBatch ? bstart[lo + 1] : 0;
      const L v0 = bsv[lo], v1 = lo + 1 < kBatch ? bsv[lo + 1] : L(0);
#pragma unroll
      for (int u = 0; u < kPV; ++u) {
        const long long slot = wbase + u * 32 + lane;
        ok[u] = slot < total;
        const bool second = slot >= x1;
        e[u] = second ? s1 + (slot - x1) : s0 + (slot - x0);
        sv[u] = second ? v1 : v0;
      }
    };
    int64_t e[kPV];
    bool ok0[kPV], ok1[kPV];
    L sv0[kPV], sv1[kPV];
    uint32_t d0[kPV], d1[kPV];
    W w0[kPV], w1[kPV];
    slots(0, e, ok0, sv0);
    op.fetch(a, e, ok0, d0, w0);
    for (long long b = 0; b < total; b += step) {
      const bool more = b + step < total;
      if (more) {
        slots(b + step, e, ok1, sv1);
        op.fetch(a, e, ok1, d1, w1);
      }
      if (a.cta_edges) my_proc += count_ok(ok0);
      op.apply(d0, w0, sv0, ok0);
#pragma unroll
      for (int u = 0; u < kPV; ++u) d0[u] = d1[u], w0[u] = w1[u], sv0[u] = sv1[u], ok0[u] = more && ok1[u];
    }
    __syncthreads();
  }
  cta_flush(a, my_proc, ctl->round);
}

// ---- cc round 0 as one stream over the edges.  Round 0 of cc has every
// vertex in the frontier and every label equal to its id (apps.py:114-127),
// so the round's push relaxations lab[v] = min(lab[v], u) over the
// symmetrized edges (u, v) are, per row, new[v] = min(v, min of the row's
// ids): one pass streaming the column ids and their row ids (Graph::sym_src)
// of the graph in its original numbering -- every edge is read, no label
// gather, one atomic per row run (results go into the kernel layout through
// inv).  Changed vertices set their next-frontier bit; the compaction and the
// advance kernel then close round 0 exactly as after the push kernels (same
// labels, same round log: frontier V, every edge, the reference's bins).
namespace {  // non-template kernels: one copy per translation unit
struct CcDenseArgs {
  const int64_t *off;   // original-numbering symmetrized rows
  const uint32_t *col;
  const uint32_t *src;  // row of every edge (Graph::sym_src)
  int64_t nv, ne;
  const uint32_t *inv;  // original -> kernel-layout id (nullptr: the same numbering)
  uint32_t *lab;        // kernel-layout labels, initialised to the original ids
  uint32_t *nb;         // next-frontier bitmap (kernel layout)
  Ctl *ctl;
  int64_t thr;          // huge threshold (round-log bins)
};
constexpr int kDenseV = 8;  // edges per lane in flight

// the edges as one stream (col, src): a warp takes tiles of 32 x kDenseV
// consecutive edges.  Per instruction, lanes of one row (a contiguous run)
// reduce with match.any + redux.sync.min and the run's first lane applies the
// minimum (atomicMin -- a row may continue in other instructions -- and the
// next-frontier bit when it beats the id).  A hub row spans thousands of
// instructions: the label is read first (L2) and the atomic skipped when it
// cannot lower it (a stale read is only ever too high: never a lost update;
// the bit was set by whoever lowered the label).
__device__ __forceinline__ void cc_dense_apply(const CcDenseArgs &a, uint32_t r, uint32_t m) {
  if (r == 0xffffffffu || m >= r) return;
  const uint32_t i = a.inv ? a.inv[r] : r;
  if (__ldcg(a.lab + i) <= m) return;
  atomicMin(a.lab + i, m);
  atomicOr(a.nb + (i >> 5), 1u << (i & 31u));
}
__global__ void __launch_bounds__(kTB) k_cc_dense(CcDenseArgs a) {
  const int64_t W = (int64_t)grid_warps(), step = 32 * kDenseV;
  const uint32_t lane = lane_id();
  for (int64_t b = (int64_t)global_warp() * step; b < a.ne; b += W * step) {
    uint32_t u[kDenseV], r[kDenseV];
#pragma unroll
    for (int k = 0; k < kDenseV; ++k) {
      const int64_t e = b + k * 32 + lane;
      u[k] = e < a.ne ? ld_stream(a.col + e) : 0xffffffffu;
      r[k] = e < a.ne ? ld_stream(a.src + e) : 0xffffffffu;
    }
#pragma unroll
    for (int k = 0; k < kDenseV; ++k) {
      const uint32_t grp = __match_any_sync(kFull, r[k]);
      const uint32_t m = __reduce_min_sync(grp, u[k]);
      if ((int)lane == __ffs(grp) - 1) cc_dense_apply(a, r[k], m);
    }
  }
}

// the round log of the dense round: every row is in the frontier; the
// reference's bins by degree (schedulers.py:144-167)
__global__ void __launch_bounds__(kTB) k_cc_dense_bins(CcDenseArgs a) {
  __shared__ unsigned long long red[32];
  unsigned long long hedges = 0, ledges = 0, nh = 0, nl = 0;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.nv; v += st) {
    const int64_t deg = a.off[v + 1] - a.off[v];
    const bool huge = deg >= a.thr, large = !huge && deg >= (int64_t)kLarge;
    nh += huge, nl += large;
    if (huge) hedges += (unsigned long long)deg;
    if (large) ledges += (unsigned long long)deg;
  }
  unsigned long long x = block_sum(hedges, red);
  if (threadIdx.x == 0 && x) atomicAdd(&a.ctl->huge_edges, x);
  x = block_sum(ledges, red);
  if (threadIdx.x == 0 && x) atomicAdd(&a.ctl->large_edges, x);
  x = block_sum(nh, red);
  if (threadIdx.x == 0 && x) atomicAdd(&a.ctl->nhuge, (uint32_t)x);
  x = block_sum(nl, red);
  if (threadIdx.x == 0 && x) atomicAdd(&a.ctl->nlarge, (uint32_t)x);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&a.ctl->edges, (unsigned long long)a.ne);
}
}  // namespace

// ---- CTA bin with 128-bit adjacency loads (SG_LARGE_VEC): lane l takes the
// kPV = 4 CONSECUTIVE slots 4l..4l+3 of the warp's 128-slot step, so when they
// lie in one row at a 16-byte aligned offset the column ids (and u32 weights)
// come in one ld.global.nc.v4 each instead of four scalar loads.
__device__ __forceinline__ uint4 ld_stream_v4(const uint32_t *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(l2_evict_first()));
  return v;
}

template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_large_vec(PushArgs a, Op op) {
  static_assert(kPV == 4, "k_bm_large_vec: four consecutive slots per lane");
  pdl_wait();
  pdl_trigger();
  using L = typename Op::L;
  using W = typename Op::W;
  constexpr bool kW32 = std::is_same<W, uint32_t>::value && !std::is_same<Op, BmBfs>::value;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  if (a.prefix_in_large && blockIdx.x == 0 && ctl->nhuge) huge_prefix_cta(a, op);
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  __shared__ int64_t bstart[kBatch];
  __shared__ long long bexcl[kBatch + 1];
  __shared__ L bsv[kBatch];
  __shared__ uint32_t bhead;
  const uint32_t nb = (n + kBatch - 1) / kBatch;
  const long long wstep = 32 * kPV, step = (long long)kTB * kPV;
  const uint32_t lane = threadIdx.x & 31u;
  const long long woff = (long long)(threadIdx.x >> 5) * wstep;
  const uint32_t *w32 = nullptr;
  if constexpr (kW32) w32 = op.w32;
  bool first_grab = true;
  for (;;) {
    if (threadIdx.x == 0) bhead = cta_grab(&ctl->large_head, first_grab);
    __syncthreads();
    const uint32_t bidx = bhead;
    if (bidx >= nb) break;
    if (threadIdx.x < 32) {
      const uint32_t i = bidx + threadIdx.x * nb;  // degree-mixed batch
      long long d = 0;
      if (threadIdx.x < kBatch && i < n) {
        const uint32_t v = a.largeq[i];
        const int64_t s = a.off[v];
        d = a.off[v + 1] - s;
        bstart[threadIdx.x] = s;
        bsv[threadIdx.x] = (L)a.largesv[i];
      }
      const long long incl = warp_incl_scan(d);
      if (threadIdx.x < kBatch) bexcl[threadIdx.x + 1] = incl;
      if (threadIdx.x == 0) bexcl[0] = 0;
    }
    __syncthreads();
    const long long total = bexcl[kBatch];
    // lane-contiguous slots: 4 lane + u; a warp step spans <= 2 batch vertices
    auto fetch = [&](long long b, bool (&ok)[kPV], L (&sv)[kPV], uint32_t (&d)[kPV], W (&w)[kPV]) {
      const long long wbase = b + woff;
      uint32_t lo = 0;
#pragma unroll
      for (uint32_t st = kBatch / 2; st; st >>= 1) lo = bexcl[lo + st] <= wbase ? lo + st : lo;
      const long long x0 = bexcl[lo], x1 = bexcl[lo + 1];
      const int64_t s0 = bstart[lo], s1 = lo + 1 < kBatch ? bstart[lo + 1] : 0;
      const L v0 = bsv[lo], v1 = lo + 1 < kBatch ? bsv[lo + 1] : L(0);
      int64_t e[kPV];
#pragma unroll
      for (int u = 0; u < kPV; ++u) {
        const long long slot = wbase + 4 * lane + u;
        ok[u] = slot < total;
        const bool second = slot >= x1;
        e[u] = second ? s1 + (slot - x1) : s0 + (slot - x0);
        sv[u] = second ? v1 : v0;
      }
      if (ok[3] && e[3] == e[0] + 3 && (e[0] & 3) == 0) {  // one row, aligned: 128-bit
        const uint4 c = ld_stream_v4(a.col + e[0]);
        d[0] = c.x, d[1] = c.y, d[2] = c.z, d[3] = c.w;
        if constexpr (kW32) {
          if (w32) {
            const uint4 x = ld_stream_v4(w32 + e[0]);
            w[0] = x.x, w[1] = x.y, w[2] = x.z, w[3] = x.w;
          } else {
            w[0] = w[1] = w[2] = w[3] = 1u;
          }
        } else {
#pragma unroll
          for (int u = 0; u < kPV; ++u) w[u] = (W)1;
        }
      } else {
        op.fetch(a, e, ok, d, w);
      }
    };
    bool ok0[kPV], ok1[kPV];
    L sv0[kPV], sv1[kPV];
    uint32_t d0[kPV], d1[kPV];
    W w0[kPV], w1[kPV];
    fetch(0, ok0, sv0, d0, w0);
    for (long long b = 0; b < total; b += step) {
      const bool more = b + step < total;
      if (more) fetch(b + step, ok1, sv1, d1, w1);
      if (a.cta_edges) my_proc += count_ok(ok0);
      op.apply(d0, w0, sv0, ok0);
#pragma unroll
      for (int u = 0; u < kPV; ++u) d0[u] = d1[u], w0[u] = w1[u], sv0[u] = sv1[u], ok0[u] = more && ok1[u];
    }
    __syncthreads();
  }
  cta_flush(a, my_proc, ctl->round);
}

// ---- CTA bin with the adjacency staged through shared memory.  Each lane
// issues cp.async copies of its slots' column ids (and u32 weights) for the
// step kStage - 1 ahead into a per-warp ring, so kStage - 1 steps of
// adjacency are in flight without holding registers (the register-prefetch
// loop above keeps one step); the gathers and reductions of a step read the
// staged ids.  SG_LARGE_STAGE selects it (bm_round); measured in profiles/.
#ifndef SG_STAGE_DEPTH
#define SG_STAGE_DEPTH 3
#endif
constexpr int kStage = SG_STAGE_DEPTH;
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool pred) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = pred ? 4 : 0;  // src-size 0: zero-fill, no global access
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_large_staged(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
  using L = typename Op::L;
  using W = typename Op::W;
  constexpr bool kW32 = std::is_same<W, uint32_t>::value && !std::is_same<Op, BmBfs>::value;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  if (a.prefix_in_large && blockIdx.x == 0 && ctl->nhuge) huge_prefix_cta(a, op);
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  __shared__ int64_t bstart[kBatch];
  __shared__ long long bexcl[kBatch + 1];
  __shared__ L bsv[kBatch];
  __shared__ uint32_t bhead;
  __shared__ uint32_t scol[kWarpsTB][kStage][kPV][32];
  __shared__ uint32_t sw[kW32 ? kWarpsTB : 1][kStage][kPV][32];
  const uint32_t nb = (n + kBatch - 1) / kBatch;
  const long long wstep = 32 * kPV, step = (long long)kTB * kPV;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const long long woff = (long long)warp * wstep;
  const uint32_t *w32 = nullptr;
  if constexpr (kW32) w32 = op.w32;
  bool first_grab = true;
  for (;;) {
    if (threadIdx.x == 0) bhead = cta_grab(&ctl->large_head, first_grab);
    __syncthreads();
    const uint32_t bidx = bhead;
    if (bidx >= nb) break;
    if (threadIdx.x < 32) {
      const uint32_t i = bidx + threadIdx.x * nb;  // degree-mixed batch
      long long d = 0;
      if (threadIdx.x < kBatch && i < n) {
        const uint32_t v = a.largeq[i];
        const int64_t s = a.off[v];
        d = a.off[v + 1] - s;
        bstart[threadIdx.x] = s;
        bsv[threadIdx.x] = (L)a.largesv[i];
      }
      const long long incl = warp_incl_scan(d);
      if (threadIdx.x < kBatch) bexcl[threadIdx.x + 1] = incl;
      if (threadIdx.x == 0) bexcl[0] = 0;
    }
    __syncthreads();
    const long long total = bexcl[kBatch];
    const long long nsteps = (total + step - 1) / step;
    auto slots = [&](long long b, int64_t (&e)[kPV], bool (&ok)[kPV], L (&sv)[kPV]) {
      const long long wbase = b + woff;
      uint32_t lo = 0;
#pragma unroll
      for (uint32_t st = kBatch / 2; st; st >>= 1) lo = bexcl[lo + st] <= wbase ? lo + st : lo;
      const long long x0 = bexcl[lo], x1 = bexcl[lo + 1];
      const int64_t s0 = bstart[lo], s1 = lo + 1 < kBatch ? bstart[lo + 1] : 0;
      const L v0 = bsv[lo], v1 = lo + 1 < kBatch ? bsv[lo + 1] : L(0);
#pragma unroll
      for (int u = 0; u < kPV; ++u) {
        const long long slot = wbase + u * 32 + lane;
        ok[u] = slot < total;
        const bool second = slot >= x1;
        e[u] = second ? s1 + (slot - x1) : s0 + (slot - x0);
        sv[u] = second ? v1 : v0;
      }
    };
    auto stage = [&](long long k) {  // step k's adjacency -> ring slot k % kStage
      int64_t e[kPV];
      bool ok[kPV];
      L sv[kPV];
      if (k < nsteps) slots(k * step, e, ok, sv);
      const int r = (int)(k % kStage);
#pragma unroll
      for (int u = 0; u < kPV; ++u) {
        const bool p = k < nsteps && ok[u];
        cp_async4(&scol[warp][r][u][lane], a.col + (p ? e[u] : 0), p);
        if constexpr (kW32)
          if (w32) cp_async4(&sw[warp][r][u][lane], w32 + (p ? e[u] : 0), p);
      }
      cp_async_commit();  // one group per step (empty past the end: keeps the count)
    };
#pragma unroll
    for (int k = 0; k < kStage - 1; ++k) stage(k);
    for (long long k = 0; k < nsteps; ++k) {
      stage(k + kStage - 1);
      cp_async_wait<kStage - 1>();  // step k's group has landed (this lane's own copies)
      int64_t e[kPV];
      bool ok[kPV];
      L sv[kPV];
      slots(k * step, e, ok, sv);
      const int r = (int)(k % kStage);
      uint32_t d[kPV];
      W w[kPV];
#pragma unroll
      for (int u = 0; u < kPV; ++u) {
        d[u] = scol[warp][r][u][lane];
        if constexpr (kW32) w[u] = w32 ? sw[warp][r][u][lane] : 1u;
        else w[u] = (W)1;
      }
      if (a.cta_edges) my_proc += count_ok(ok);
      op.apply(d, w, sv, ok);
    }
    cp_async_wait<0>();
    __syncthreads();
  }
  cta_flush(a, my_proc, ctl->round);
}

// Classic TWC CTA bin (Merrill; the reference's twc_kernel maps each large
// vertex to one CTA, _kernels_py.py:140-146): a CTA takes one vertex at a time
// and strides over its edges.  Used for the TWC-only ablation
// (SG_FLAG_TWC_CLASSIC); one huge vertex pins one CTA for its whole degree.
template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_large_classic(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
  using L = typename Op::L;
  __shared__ uint32_t item;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  if (a.prefix_in_large && blockIdx.x == 0 && ctl->nhuge) huge_prefix_cta(a, op);
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  bool first_grab = true;
  for (;;) {
    if (threadIdx.x == 0) item = cta_grab(&ctl->large_head, first_grab);
    __syncthreads();
    const uint32_t idx = item;
    __syncthreads();
    if (idx >= n) break;
    const uint32_t v = a.largeq[idx];
    const int64_t s = a.off[v], deg = a.off[v + 1] - s;
    const L sv = (L)a.largesv[idx];
    for (int64_t b = 0; b < deg; b += kTB * kV) {
      int64_t e[kV];
      bool ok[kV];
      L svs[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int64_t slot = b + u * kTB + threadIdx.x;
        ok[u] = slot < deg;
        e[u] = s + slot;
        svs[u] = sv;
      }
      if (a.cta_edges) my_proc += count_ok(ok);
      op.relax(a, e, ok, svs);
    }
  }
  cta_flush(a, my_proc, ctl->round);
}

// ALB huge-vertex kernel (Algorithm 2): every thread of every CTA walks the
// huge edges cyclically (g = p*T + tid) or blocked (g = tid*ceil(e/T) + p)
template <class Op, bool BLOCKED>
__global__ void __launch_bounds__(kTB) k_bm_lb(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
  using L = typename Op::L;
  __shared__ int64_t spre[kHugeSmem], sstart[kHugeSmem];
  __shared__ unsigned long long sval[kHugeSmem];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t nh = ctl->nhuge;
  if (!nh) return;
  const int64_t E = (int64_t)ctl->huge_edges;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  const int64_t T = (int64_t)gridDim.x * kTB;
  const int64_t tid = (int64_t)blockIdx.x * kTB + threadIdx.x;
  const int64_t passes = (E + T - 1) / T;
  if (!BLOCKED && a.threshold >= 32 * kV * kLBSteps) {
    // cyclic at warp granularity: warp w takes the CH consecutive edge ids of
    // chunks w, w + W, w + 2W, ... (consecutive lanes still read consecutive
    // adjacency entries, the point of the paper's cyclic distribution).
    // Every huge vertex owns >= threshold >= CH edges, so a chunk spans at
    // most two of them: find_owner (worklist.py:96-119) is one warp-uniform
    // two-level bisection per chunk, amortised over kLBSteps relax steps.
    constexpr int64_t CH = 32 * kV * kLBSteps;
    const int64_t nwarps = T >> 5, nch = (E + CH - 1) / CH;
    const uint32_t lane = lane_id();
    const Coarse cx = coarse_build(spre, a.hpre, nh);  // spre: >= kCoarse entries
    for (int64_t c = tid >> 5; c < nch; c += nwarps) {
      const int64_t g0 = c * CH;
      const uint32_t o = cx.find(g0);
      const int64_t x0 = o ? a.hpre[o - 1] : 0, x1 = a.hpre[o];
      const int64_t s0 = a.hstart[o], s1 = o + 1 < nh ? a.hstart[o + 1] : 0;
      const L v0 = (L)a.hval[o], v1 = o + 1 < nh ? (L)a.hval[o + 1] : L(0);
      for (int st = 0; st < kLBSteps; ++st) {
        const int64_t gs = g0 + (int64_t)st * 32 * kV;
        if (gs >= E) break;
        int64_t e[kV];
        bool ok[kV];
        L sv[kV];
#pragma unroll
        for (int u = 0; u < kV; ++u) {
          const int64_t g = gs + u * 32 + lane;
          ok[u] = g < E;
          const bool second = g >= x1;
          e[u] = second ? s1 + (g - x1) : s0 + (g - x0);
          sv[u] = second ? v1 : v0;
        }
        if (a.cta_edges) my_proc += count_ok(ok);
        op.relax(a, e, ok, sv);
      }
    }
    cta_flush(a, my_proc, ctl->round);
    return;
  }
  const bool staged = nh <= kHugeSmem;
  if (staged) {
    for (uint32_t i = threadIdx.x; i < nh; i += kTB)
      spre[i] = a.hpre[i], sstart[i] = a.hstart[i], sval[i] = a.hval[i];
    __syncthreads();
  }
  for (int64_t p0 = 0; p0 < passes; p0 += kV) {
    int64_t e[kV];
    bool ok[kV];
    L sv[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t p = p0 + u;
      const int64_t g = BLOCKED ? tid * passes + p : p * T + tid;
      ok[u] = p < passes && g < E;
      const int64_t gg = ok[u] ? g : 0;
      if (staged) {  // find_owner (worklist.py:96-119) over the staged prefix
        const uint32_t o = owner_search(spre, nh, gg);
        e[u] = sstart[o] + (gg - (o ? spre[o - 1] : 0));
        sv[u] = (L)sval[o];
      } else {
        const uint32_t o = owner_search(a.hpre, nh, gg);
        e[u] = a.hstart[o] + (gg - (o ? a.hpre[o - 1] : 0));
        sv[u] = (L)a.hval[o];
      }
    }
    if (a.cta_edges) my_proc += count_ok(ok);
    op.relax(a, e, ok, sv);
  }
  cta_flush(a, my_proc, ctl->round);
}

// ------------------------------------------- the other schedulers (run level)
// vertex (_kernels_py.py:88-97): frontier vertex i -> one thread, which walks
// all of its edges (no balancing: the baseline the bins exist to beat)
template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_vertex(PushArgs a, Op op) {
  using L = typename Op::L;
  __shared__ unsigned long long red[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  const Src src = resolve_src(a, ctl);
  unsigned long long my_edges = 0;
  const uint64_t st = (uint64_t)gridDim.x * kTB;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kTB; i0 < src.n; i0 += st) {
    const uint64_t i = i0 + threadIdx.x;
    int64_t s = 0, deg = 0;
    L sv = 0;
    if (i < src.n) {
      const uint32_t v = src.at(i);
      s = a.off[v];
      deg = a.off[v + 1] - s;
      sv = op.src_val(i, v);
    }
    my_edges += (unsigned long long)deg;
    for (int64_t j = 0; j < deg; j += kV) {
      int64_t e[kV];
      bool ok[kV];
      L svs[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) ok[u] = j + u < deg, e[u] = s + j + u, svs[u] = sv;
      if (a.cta_edges) my_proc += count_ok(ok);
      op.relax(a, e, ok, svs);
    }
  }
  const unsigned long long bs = block_sum(my_edges, red);
  if (threadIdx.x == 0 && bs) atomicAdd(&ctl->edges, bs);
  cta_flush(a, my_proc, ctl->round);
}

// lb / edge: the whole frontier as one prefix-summed list (PrefixWork over
// every active vertex, schedulers.py:280-283), built by a multi-CTA scan in
// tiles of kFT entries: hugeq / hstart / hval / hpre as for ALB's huge bin
constexpr int kFT = 1024;
template <class Op>
__global__ void __launch_bounds__(kTB) k_front_tiles(PushArgs a, Op op, long long *tsum) {
  __shared__ long long red[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  op.begin(ctl->round);
  const Src src = resolve_src(a, ctl);
  const uint32_t ntiles = (src.n + kFT - 1) / kFT;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    long long sum = 0;
#pragma unroll
    for (int k = 0; k < kFT / kTB; ++k) {
      const uint64_t i = (uint64_t)t * kFT + k * kTB + threadIdx.x;
      if (i < src.n) {
        const uint32_t v = src.at(i);
        const int64_t s = a.off[v], d = a.off[v + 1] - s;
        a.hugeq[i] = v;
        a.hstart[i] = s;
        a.hval[i] = (unsigned long long)op.src_val(i, v);
        a.hpre[i] = d;  // degrees; k_front_apply turns them into the inclusive prefix
        sum += d;
      }
    }
    sum = block_sum(sum, red);
    if (threadIdx.x == 0) tsum[t] = sum;
    __syncthreads();
  }
}
// exclusive scan of the tile sums (one CTA); totals into Ctl
static __global__ void __launch_bounds__(1024) k_front_scan(PushArgs a, long long *tsum) {
  __shared__ long long red[32];
  __shared__ long long carry;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const Src src = resolve_src(a, ctl);
  const uint32_t ntiles = (src.n + kFT - 1) / kFT;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < ntiles; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    const long long d = i < ntiles ? tsum[i] : 0;
    const long long x = warp_incl_scan(d);
    if (lane_id() == 31) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) red[threadIdx.x] = warp_incl_scan(red[threadIdx.x]);
    __syncthreads();
    const long long incl = carry + ((threadIdx.x >> 5) ? red[(threadIdx.x >> 5) - 1] : 0) + x;
    if (i < ntiles) tsum[i] = incl - d;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ctl->huge_edges = (unsigned long long)carry;
    ctl->edges = (unsigned long long)carry;
    ctl->nhuge = src.n;
  }
}
static __global__ void __launch_bounds__(kTB) k_front_apply(PushArgs a, const long long *tsum) {
  __shared__ long long red[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const Src src = resolve_src(a, ctl);
  const uint32_t ntiles = (src.n + kFT - 1) / kFT;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    long long carry = tsum[t];
#pragma unroll
    for (int k = 0; k < kFT / kTB; ++k) {
      const uint64_t i = (uint64_t)t * kFT + k * kTB + threadIdx.x;
      const long long d = i < src.n ? a.hpre[i] : 0;
      const long long x = warp_incl_scan(d);
      if (lane_id() == 31) red[threadIdx.x >> 5] = x;
      __syncthreads();
      long long wpre = 0, tot = 0;
      for (int w = 0; w < kWarpsTB; ++w) {
        if (w < (int)(threadIdx.x >> 5)) wpre += red[w];
        tot += red[w];
      }
      if (i < src.n) a.hpre[i] = carry + wpre + x;
      carry += tot;
      __syncthreads();
    }
  }
}

// edge (_kernels_py.py:100-117): thread t takes the contiguous active-edge
// range [t*chunk, (t+1)*chunk); the owner is found once and then walked
// forward (the O(1) endpoint step the reference gets from its COO array)
template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_edge(PushArgs a, Op op) {
  using L = typename Op::L;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t nh = ctl->nhuge;
  const int64_t E = (int64_t)ctl->huge_edges;
  if (!nh || !E) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  const int64_t T = (int64_t)gridDim.x * kTB;
  const int64_t tid = (int64_t)blockIdx.x * kTB + threadIdx.x;
  const int64_t chunk = (E + T - 1) / T;
  const int64_t g0 = tid * chunk, g1 = min(g0 + chunk, E);
  if (g0 >= E) return;
  uint32_t o = owner_search(a.hpre, nh, g0);
  for (int64_t g = g0; g < g1; g += kV) {
    int64_t e[kV];
    bool ok[kV];
    L sv[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t gg = g + u;
      ok[u] = gg < g1;
      while (ok[u] && gg >= a.hpre[o]) ++o;
      e[u] = a.hstart[o] + (gg - (o ? a.hpre[o - 1] : 0));
      sv[u] = (L)a.hval[o];
    }
    if (a.cta_edges) my_proc += count_ok(ok);
    op.relax(a, e, ok, sv);
  }
  cta_flush(a, my_proc, ctl->round);
}

// next frontier from the round's bitmap: ids ascending within each warp's
// 1024-vertex range, one atomic per warp range, coalesced id / snapshot writes
template <class Op>
__global__ void __launch_bounds__(kTB) k_bm_compact(PushArgs a, Op op) {
  pdl_wait();
  pdl_trigger();
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  op.begin(ctl->round);
  const uint32_t nwords = (a.nv + 31) / 32, lane = lane_id();
  const uint32_t warps = (gridDim.x * kTB) >> 5;
  uint32_t *q = a.q[0];
  // warp-major over CTAs: consecutive 32-word blocks go to different CTAs
  // (SMs), so a dense run of frontier bits -- the relabeled hot set -- is
  // spread over the chip instead of the first few CTAs
  const uint32_t gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  for (uint32_t w0 = gw * 32; w0 < nwords; w0 += warps * 32) {
    const uint32_t wi = w0 + lane;
    uint32_t bits = wi < nwords ? op.take(wi) : 0u;
    if (bits && wi * 32u + 31u >= a.zlo) {  // members without out-edges: count, do not queue
      const uint32_t keep = wi * 32u >= a.zlo ? 0u : (1u << (a.zlo - wi * 32u)) - 1u;
      uint32_t z = bits & ~keep;
      bits &= keep;
      if (z) atomicAdd(&ctl->nzero, (uint32_t)__popc(z));
      while (z) {
        const uint32_t b = __ffs(z) - 1;
        z &= z - 1;
        op.emit_zero(wi * 32u + b);
      }
    }
    const uint32_t cnt = __popc(bits);
    const uint32_t incl = warp_incl_scan(cnt);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (!total) continue;
    uint32_t pos0 = 0;
    if (lane == 0) pos0 = atomicAdd(&ctl->nsize, total);
    pos0 = __shfl_sync(kFull, pos0, 0);
    const uint32_t excl = incl - cnt;
    // 4 emits per lane in flight: a dense word block (up to 1024 vertices,
    // clustered at low ids on the relabeled store) is 8 steps, not 32
    // dependent load -> store chains
    constexpr int kE = 4;
    for (uint32_t k0 = 0; k0 < total; k0 += 32 * kE) {
      uint32_t v[kE];
      typename Op::E x[kE];
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const uint32_t slot = k0 + u * 32 + lane;
        const int o = warp_owner(incl, slot);
        const uint32_t bo = __shfl_sync(kFull, bits, o);
        const uint32_t eo = __shfl_sync(kFull, excl, o);
        v[u] = slot < total ? (w0 + (uint32_t)o) * 32 + __fns(bo, 0, (int)(slot - eo) + 1) : 0u;
      }
#pragma unroll
      for (int u = 0; u < kE; ++u)
        if (k0 + u * 32 + lane < total) x[u] = op.emit_load(v[u]);
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const uint32_t slot = k0 + u * 32 + lane;
        if (slot < total) {
          q[pos0 + slot] = v[u];
          op.emit_store(pos0 + slot, v[u], x[u]);
        }
      }
    }
  }
}

}  // namespace sg
