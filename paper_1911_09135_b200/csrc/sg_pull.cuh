// sg_pull.cuh — ALB pull round (pr: rank sums, kcore: surviving-neighbour counts).
//
// Reference: OP_PULL_ADD out[row] += aux[col[e]] (_kernels_py.py:73-75), rows of
// the CSC view; pr folds new = (1-d) + d*acc and stops on max|new-old| <= eps
// (apps.py:176-186); kcore counts alive neighbours of frontier vertices and
// kills those below k (apps.py:217-232).
// B200 mapping: rows are owned by exactly one lane / CTA in the TWC bins, so
// their sums are formed in registers (warp-segmented shuffle scans, CTA tree
// reduction — deterministic order) and folded in the same kernel (pr writes
// rank and next round's aux = rank*inv_outdeg; kcore emits the dying list).
// Only huge rows are split across CTAs by the LB kernel; their partial sums
// are pre-reduced per warp segment and combined with one atomicAdd per segment.
#pragma once
#include "sg_bm.cuh"

namespace sg {

#ifndef SG_PULL_V
#define SG_PULL_V 8
#endif
// edges per lane per step in the pull kernels (pr gathers 8-byte aux values:
// kcore / pr measured 7 % slower at the push kernels' kV = 6)
constexpr int kPullV = SG_PULL_V;
#ifndef SG_PULL_SEQ
#define SG_PULL_SEQ 32  // longest per-window row segment summed sequentially (0: scan only)
#endif
static_assert(kPullV * 32 <= (int)kLarge, "k_pull_large: a warp step must span <= 2 rows");


#ifndef SG_PR_UNROLL
#define SG_PR_UNROLL 4
#endif

struct PullArgs {
  const int64_t *off;
  const uint32_t *col;
  uint32_t nv;
  Ctl *ctl;
  uint32_t *q[2];  // kcore frontier queues
  uint32_t *largeq, *hugeq;
  int64_t *hpre, *hstart;
  int64_t threshold;
  int dynamic_bins;  // 1: kcore (bins found per round); 0: pr (static bins, dense rows)
  uint32_t *dying;   // kcore dying list (count ctl->ndying)
  RoundStat *stats;
  Cuts cuts;                // devices > 1: partition accounting (engine.py:215-234)
  const uint32_t *mcount;   // mirror_count per vertex (devices > 1), else nullptr
  uint32_t row_lo, row_n;   // a dense round covers rows [row_lo, row_lo + row_n)
  int vertex;               // vertex scheduler: k_pull_vertex instead of the bins
  unsigned long long *cta_edges;  // SG_FLAG_CTA_COUNTS (see PushArgs)
  uint32_t cta_g, cta_rounds;
};

// pr: acc = sum aux[u]; new = (1-d) + d*acc (two roundings, as numpy); aux' = new*inv
struct PrOp {
  using A = double;
  static constexpr bool kWarpMedium = false;  // medium rows join the segmented warp gather
  static constexpr int kUnroll = SG_PR_UNROLL;
  const double *aux0, *aux1;
  double *next0, *next1;
  double *rank;
  const double *inv;
  double d, omd;
  const uint32_t *mcount = nullptr;  // devices > 1: comm_broadcast of changed ranks
  const double *aux = nullptr;
  double *auxn = nullptr;
  double dmax = 0.0;
  unsigned long long bcast = 0;
  // source-block tiling (prep_pr): 1 first block (carry = acc), 2 middle
  // block (carry += acc), 3 last block (acc = carry + acc, then the fold)
  double *carry = nullptr;
  int tmode = 0;
  __device__ __forceinline__ void begin(uint32_t round) {
    aux = (round & 1) ? aux1 : aux0;
    auxn = (round & 1) ? next1 : next0;
  }
  __device__ __forceinline__ A load(uint32_t u) const { return __ldg(aux + u); }
  __device__ __forceinline__ bool finish(uint32_t v, A acc) {
    if (tmode == 1) {
      carry[v] = acc;
      return false;
    }
    if (tmode == 2) {
      carry[v] = carry[v] + acc;
      return false;
    }
    if (tmode == 3) acc = carry[v] + acc;
    double nw = __dadd_rn(omd, __dmul_rn(d, acc));
    const double old = rank[v];
    double dl = fabs(__dsub_rn(nw, old));
    dmax = dl > dmax ? dl : dmax;
    if (mcount && nw != old) bcast += mcount[v];  // engine.py:232-234
    rank[v] = nw;
    auxn[v] = __dmul_rn(nw, inv[v]);
    return false;
  }
};

// kcore: count = sum alive[u] with multiplicity (integers: any order is exact)
struct KcOp {
  using A = uint32_t;
  static constexpr bool kWarpMedium = true;  // TWC warp bin: one medium row per warp step
  static constexpr int kUnroll = 4;
  const uint8_t *alive;
  uint32_t k;
  double dmax = 0.0;            // unused
  unsigned long long bcast = 0;  // unused (kcore counts broadcasts at the kill)
  __device__ __forceinline__ void begin(uint32_t) {}
  __device__ __forceinline__ A load(uint32_t u) const { return alive[u]; }
  __device__ __forceinline__ bool finish(uint32_t, A acc) const { return acc < k; }
};

__device__ __forceinline__ void atomic_max_dbits(unsigned long long *p, double x) {
  atomicMax(p, (unsigned long long)__double_as_longlong(x));  // x >= 0
}

template <class Op>
__global__ void __launch_bounds__(kTB) k_pull_twc(PullArgs a, Op op) {
  __shared__ unsigned long long red[32];
  __shared__ double redd[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  unsigned long long my_proc = 0;
  const bool dense = !a.dynamic_bins || ctl->dense;
  const uint32_t n = dense ? a.row_n : ctl->fsize;
  const uint32_t *list = (round & 1) ? a.q[1] : a.q[0];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  unsigned long long my_edges = 0, my_large = 0;
  // dynamic fetch: a warp grabs kChunkGrab chunks of 32 rows at a time (the
  // dense pr rows are degree-skewed, a static split leaves a long tail)
  const uint32_t nchunks = (n + 31) / 32;
  uint32_t c = 0, c_end = 0;
  (void)warp;
  for (;;) {
    if (c == c_end) {
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
    const bool valid = i < n;
    if (valid) {
      v = dense ? a.row_lo + (uint32_t)i : list[i];
      s = a.off[v];
      deg = a.off[v + 1] - s;
    }
    my_edges += (unsigned long long)deg;
    const bool huge = deg >= a.threshold;
    const bool large = !huge && deg >= (int64_t)kLarge;
    if (a.dynamic_bins) {
      warp_append(huge, v, a.hugeq, &ctl->nhuge);
      warp_append(large, v, a.largeq, &ctl->nlarge);
      if (large) my_large += (unsigned long long)deg;
      if (a.cuts.D > 1) {  // which simulated devices launch inspect/twc and lb this round
        const uint32_t bit = valid ? 1u << owner_of(a.cuts, v) : 0u;
        const uint32_t tw = __reduce_or_sync(kFull, bit);
        const uint32_t lb = __reduce_or_sync(kFull, huge ? bit : 0u);
        if (lane == 0 && tw) atomicOr(&ctl->part_twc_mask, tw);
        if (lane == 0 && lb) atomicOr(&ctl->part_lb_mask, lb);
      }
    }
    // small rows (deg < 32): warp gather over the chunk's rows with a
    // segmented reduction; medium rows (32 <= deg < kLarge): the whole warp
    // takes one row at a time (TWC's warp bin, schedulers.py:157-159)
    const bool mine = valid && !huge && !large;
    const bool small = mine && (deg < 32 || !Op::kWarpMedium);
    const uint32_t gd = small ? (uint32_t)deg : 0u;
    const uint32_t incl = warp_incl_scan(gd);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - gd;
    typename Op::A acc = 0;
    constexpr int KP = Op::kUnroll;
#if SG_PULL_SEQ
    // short-segment windows: park the gathered values in shared memory and
    // let each owner lane sum its own segment in order -- a few shared-memory
    // wavefronts instead of the segmented scan's ~25 shuffles per 32 slots
    // (the data pipe is what bounds this kernel, ncu)
    __shared__ typename Op::A sbuf[kWarpsTB][32 * KP];
#endif
    for (uint32_t base = 0; base < total; base += 32 * KP) {
      int o[KP];
      uint32_t src[KP];
      typename Op::A x[KP];
#pragma unroll
      for (int u = 0; u < KP; ++u) {  // KP adjacency loads in flight
        const uint32_t slot = base + u * 32 + lane;
        o[u] = warp_owner(incl, slot);
        const int64_t so = shfl64(s, o[u]);
        const uint32_t eo = __shfl_sync(kFull, excl, o[u]);
        src[u] = slot < total ? ld_stream(a.col + so + (slot - eo)) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < KP; ++u) {  // then KP value gathers in flight
        x[u] = src[u] != 0xffffffffu ? op.load(src[u]) : typename Op::A(0);
        my_proc += src[u] != 0xffffffffu;
      }
#if SG_PULL_SEQ
      {
        const uint32_t wlo = excl > base ? excl : base;
        const uint32_t whi = incl < base + 32 * KP ? incl : base + 32 * KP;
        const uint32_t len = wlo < whi ? whi - wlo : 0u;
        const uint32_t maxlen = __reduce_max_sync(kFull, len);
        if (maxlen <= SG_PULL_SEQ) {
#pragma unroll
          for (int u = 0; u < KP; ++u) sbuf[warp][u * 32 + lane] = x[u];
          __syncwarp();
          typename Op::A sum = 0;
          for (uint32_t j = 0; j < maxlen; ++j)
            if (j < len) sum += sbuf[warp][wlo - base + j];
          acc += sum;
          __syncwarp();
          continue;
        }
      }
#endif
#pragma unroll
      for (int u = 0; u < KP; ++u) {
        const uint32_t cb = base + u * 32;
        // segmented inclusive scan (owners are non-decreasing along the lanes)
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          typename Op::A y = __shfl_up_sync(kFull, x[u], dd);
          int oo = __shfl_up_sync(kFull, o[u], dd);
          if (lane >= (uint32_t)dd && oo == o[u]) x[u] += y;
        }
        // each owner lane picks up the total of its segment in this chunk
        const uint32_t lo = excl > cb ? excl : cb;
        const uint32_t hi = incl < cb + 32 ? incl : cb + 32;
        typename Op::A seg = __shfl_sync(kFull, x[u], (int)((hi - 1 - cb) & 31u));
        if (lo < hi) acc += seg;
      }
    }
    uint32_t mm = __ballot_sync(kFull, mine && !small);
    while (mm) {
      const int l = __ffs(mm) - 1;
      mm &= mm - 1;
      const int64_t ms = shfl64(s, l);
      const uint32_t md = (uint32_t)__shfl_sync(kFull, (uint32_t)deg, l);
      typename Op::A x = 0;
      for (uint32_t b = 0; b < md; b += 32 * kPullV) {
        uint32_t src[kPullV];
#pragma unroll
        for (int u = 0; u < kPullV; ++u) {
          const uint32_t j = b + u * 32 + lane;
          src[u] = j < md ? ld_stream(a.col + ms + j) : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < kPullV; ++u) {
          x += src[u] != 0xffffffffu ? op.load(src[u]) : typename Op::A(0);
          my_proc += src[u] != 0xffffffffu;
        }
      }
      x = __shfl_sync(kFull, warp_sum(x), l);  // lane l's butterfly: a fixed order
      if (lane == (uint32_t)l) acc = x;
    }
    bool die = false;
    if (mine) die = op.finish(v, acc);
    warp_append(die, v, a.dying, &ctl->ndying);
  }
  if (a.dynamic_bins) {
    unsigned long long bs = block_sum(my_edges, red);
    if (threadIdx.x == 0 && bs) atomicAdd(&ctl->edges, bs);
    bs = block_sum(my_large, red);
    if (threadIdx.x == 0 && bs) atomicAdd(&ctl->large_edges, bs);
  }
  if (sizeof(typename Op::A) == 8) {
    double m = warp_max(op.dmax);
    if (lane == 0) redd[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kWarpsTB; ++w) m = redd[w] > m ? redd[w] : m;
      if (m > 0) atomic_max_dbits(&ctl->delta_bits, m);
    }
    if (a.mcount) {
      unsigned long long b = warp_sum(op.bcast);
      if (lane == 0 && b) atomicAdd(&ctl->comm_bcast, b);
    }
  }
  cta_flush(a, my_proc, ctl->round);
}

// vertex scheduler (_kernels_py.py:88-97): one thread folds one row
template <class Op>
__global__ void __launch_bounds__(kTB) k_pull_vertex(PullArgs a, Op op) {
  __shared__ unsigned long long red[32];
  __shared__ double redd[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  unsigned long long my_proc = 0;
  const bool dense = !a.dynamic_bins || ctl->dense;
  const uint32_t n = dense ? a.row_n : ctl->fsize;
  const uint32_t *list = (round & 1) ? a.q[1] : a.q[0];
  unsigned long long my_edges = 0;
  const uint64_t st = (uint64_t)gridDim.x * kTB;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kTB; i0 < n; i0 += st) {
    const uint64_t i = i0 + threadIdx.x;
    bool die = false;
    uint32_t v = 0;
    if (i < n) {
      v = dense ? a.row_lo + (uint32_t)i : list[i];
      const int64_t s = a.off[v], e = a.off[v + 1];
      my_edges += (unsigned long long)(e - s);
      my_proc += (unsigned long long)(e - s);
      typename Op::A acc = 0;
      for (int64_t j = s; j < e; j += 4) {
        typename Op::A x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = j + u < e ? op.load(a.col[j + u]) : typename Op::A(0);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += x[u];
      }
      die = op.finish(v, acc);
    }
    warp_append(die, v, a.dying, &ctl->ndying);
  }
  if (a.dynamic_bins) {
    const unsigned long long bs = block_sum(my_edges, red);
    if (threadIdx.x == 0 && bs) atomicAdd(&ctl->edges, bs);
  }
  if (sizeof(typename Op::A) == 8) {
    double m = warp_max(op.dmax);
    if (lane_id() == 0) redd[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kWarpsTB; ++w) m = redd[w] > m ? redd[w] : m;
      if (m > 0) atomic_max_dbits(&ctl->delta_bits, m);
    }
    if (a.mcount) {
      unsigned long long b = warp_sum(op.bcast);
      if (lane_id() == 0 && b) atomicAdd(&ctl->comm_bcast, b);
    }
  }
  cta_flush(a, my_proc, ctl->round);
}

// TWC CTA bin: edge-balanced batches of kBatch rows (degree-mixed, dynamic
// fetch).  Each warp takes 32*kPullV consecutive slots per step; rows own >= kLarge
// >= 32*kPullV slots, so a step spans <= 2 rows.  A warp carries one running sum
// for its current row and parks it in part[warp][row] when the row changes
// (each warp meets a row in one contiguous stretch), and the batch's rows are
// folded as part[0][r] + ... + part[7][r]: a fixed order, deterministic.
template <class Op>
__global__ void __launch_bounds__(kTB) k_pull_large(PullArgs a, Op op) {
  using A = typename Op::A;
  __shared__ int64_t bstart[kBatch];
  __shared__ long long bexcl[kBatch + 1];
  __shared__ uint32_t brow[kBatch];
  __shared__ A part[kWarpsTB][kBatch];
  __shared__ uint32_t bhead;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t nb = (n + kBatch - 1) / kBatch;
  for (;;) {
    if (threadIdx.x == 0) bhead = atomicAdd(&ctl->large_head, 1u);
    for (uint32_t i = threadIdx.x; i < kWarpsTB * kBatch; i += kTB) part[i / kBatch][i % kBatch] = A(0);
    __syncthreads();
    const uint32_t bidx = bhead;
    if (bidx >= nb) break;
    if (warp == 0) {
      const uint32_t i = bidx + lane * nb;  // degree-mixed batch
      long long d = 0;
      uint32_t v = 0;
      if (lane < kBatch && i < n) {
        v = a.largeq[i];
        const int64_t s0 = a.off[v];
        d = a.off[v + 1] - s0;
        bstart[lane] = s0;
      }
      if (lane < kBatch) brow[lane] = v;
      const long long incl = warp_incl_scan(d);
      if (lane < kBatch) bexcl[lane + 1] = incl;
      if (lane == 0) bexcl[0] = 0;
    }
    __syncthreads();
    const long long total = bexcl[kBatch];
    int cur_o = -1;
    A cur = 0;
    for (long long b = 0; b < total; b += kTB * kPullV) {
      const long long wbase = b + (long long)warp * (32 * kPullV);
      if (wbase >= total) continue;
      uint32_t lo = 0;  // last o with bexcl[o] <= wbase
#pragma unroll
      for (uint32_t step = kBatch / 2; step; step >>= 1)
        lo = bexcl[lo + step] <= wbase ? lo + step : lo;
      const long long x0 = bexcl[lo], x1 = bexcl[lo + 1];
      const int64_t s0 = bstart[lo], s1 = lo + 1 < kBatch ? bstart[lo + 1] : 0;
      uint32_t src[kPullV];
      bool sec[kPullV];
#pragma unroll
      for (int u = 0; u < kPullV; ++u) {
        const long long slot = wbase + u * 32 + lane;
        sec[u] = slot >= x1;
        src[u] = slot < total ? ld_stream(a.col + (sec[u] ? s1 + (slot - x1) : s0 + (slot - x0)))
                              : 0xffffffffu;
      }
      A xa = 0, xb = 0;
#pragma unroll
      for (int u = 0; u < kPullV; ++u) {
        const A y = src[u] != 0xffffffffu ? op.load(src[u]) : A(0);
        my_proc += src[u] != 0xffffffffu;
        if (sec[u]) xb += y;
        else xa += y;
      }
      xa = __shfl_sync(kFull, warp_sum(xa), 0);  // lane 0's butterfly: fixed order
      xb = __shfl_sync(kFull, warp_sum(xb), 0);
      if ((int)lo != cur_o) {
        if (cur_o >= 0 && lane == 0) part[warp][cur_o] = cur;
        cur_o = (int)lo;
        cur = 0;
      }
      cur += xa;
      if (x1 < wbase + 32 * kPullV && x1 < total) {  // the step crossed into row lo + 1
        if (lane == 0) part[warp][cur_o] = cur;
        cur_o = (int)lo + 1;
        cur = xb;
      }
    }
    if (cur_o >= 0 && lane == 0) part[warp][cur_o] = cur;
    __syncthreads();
    if (warp == 0) {
      A acc = 0;
#pragma unroll
      for (int w = 0; w < kWarpsTB; ++w) acc += part[w][lane];
      const bool row = lane < kBatch && bidx + lane * nb < n;
      const bool die = row && op.finish(brow[lane], acc);
      warp_append(die, brow[lane], a.dying, &ctl->ndying);
    }
    __syncthreads();
  }
  if (warp == 0) {
    if (sizeof(A) == 8) {
      const double m = warp_max(op.dmax);
      if (lane == 0 && m > 0) atomic_max_dbits(&ctl->delta_bits, m);
    }
    const unsigned long long bc = warp_sum(op.bcast);
    if (lane == 0 && bc) atomicAdd(&ctl->comm_bcast, bc);
  }
  cta_flush(a, my_proc, ctl->round);
}

// Classic TWC CTA bin for the TWC-only ablation (SG_FLAG_TWC_CLASSIC): one
// CTA per row (dynamic fetch), block tree reduction
template <class Op>
__global__ void __launch_bounds__(kTB) k_pull_large_classic(PullArgs a, Op op) {
  using A = typename Op::A;
  __shared__ A red[32];
  __shared__ uint32_t item;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  for (;;) {
    if (threadIdx.x == 0) item = atomicAdd(&ctl->large_head, 1u);
    __syncthreads();
    const uint32_t idx = item;
    __syncthreads();
    if (idx >= n) break;
    const uint32_t v = a.largeq[idx];
    const int64_t s = a.off[v], e = a.off[v + 1];
    A x = 0;
    for (int64_t b = s + threadIdx.x; b < e; b += kTB * kPullV) {
      uint32_t src[kPullV];
#pragma unroll
      for (int u = 0; u < kPullV; ++u) src[u] = b + u * kTB < e ? ld_stream(a.col + b + u * kTB) : 0xffffffffu;
#pragma unroll
      for (int u = 0; u < kPullV; ++u) {
        x += src[u] != 0xffffffffu ? op.load(src[u]) : A(0);
        my_proc += src[u] != 0xffffffffu;
      }
    }
    x = block_sum(x, red);
    if (threadIdx.x == 0 && op.finish(v, x)) a.dying[atomicAdd(&ctl->ndying, 1u)] = v;
  }
  if (sizeof(A) == 8 && threadIdx.x == 0 && op.dmax > 0) atomic_max_dbits(&ctl->delta_bits, op.dmax);
  if (threadIdx.x == 0 && op.bcast) atomicAdd(&ctl->comm_bcast, op.bcast);
  cta_flush(a, my_proc, ctl->round);
}

// PrefixWork of the huge rows (no labels needed for pull)
static __global__ void __launch_bounds__(1024) k_pull_prefix(PullArgs a) {
  __shared__ long long red[32];
  __shared__ long long carry;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t n = ctl->nhuge;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < n; b += 1024) {
    uint32_t i = b + threadIdx.x;
    long long d = 0;
    if (i < n) {
      uint32_t v = a.hugeq[i];
      a.hstart[i] = a.off[v];
      d = a.off[v + 1] - a.off[v];
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

// huge rows: cyclic / blocked over all threads, warp-segmented pre-reduction
template <class Op, bool BLOCKED>
__global__ void __launch_bounds__(kTB) k_pull_lb(PullArgs a, Op op, typename Op::A *hacc) {
  __shared__ int64_t spre[kHugeSmem];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t nh = ctl->nhuge;
  if (!nh) return;
  op.begin(ctl->round);
  unsigned long long my_proc = 0;
  const int64_t E = (int64_t)ctl->huge_edges;
  const int64_t *pre = a.hpre;
  if (nh <= kHugeSmem) {
    for (uint32_t i = threadIdx.x; i < nh; i += kTB) spre[i] = a.hpre[i];
    __syncthreads();
    pre = spre;
  }
  const uint32_t lane = lane_id();
  const int64_t T = (int64_t)gridDim.x * kTB;
  const int64_t tid = (int64_t)blockIdx.x * kTB + threadIdx.x;
  const int64_t passes = (E + T - 1) / T;
  if (!BLOCKED && a.threshold >= 32 * kPullV) {
    // warp-granular cyclic chunks of 32*kPullV edge ids, spanning <= 2 huge rows:
    // one warp-uniform find_owner per chunk, two warp sums, <= 2 atomics
    constexpr int64_t CH = 32 * kPullV;
    const int64_t nwarps = T >> 5, nch = (E + CH - 1) / CH;
    __shared__ int64_t csample[kCoarse];
    const Coarse cx = coarse_build(csample, a.hpre, nh);
    for (int64_t c = tid >> 5; c < nch; c += nwarps) {
      const int64_t g0 = c * CH;
      const uint32_t o = cx.find(g0);
      const int64_t x0 = o ? a.hpre[o - 1] : 0, x1 = a.hpre[o];
      const int64_t s0 = a.hstart[o], s1 = o + 1 < nh ? a.hstart[o + 1] : 0;
      uint32_t src[kPullV];
      bool sec[kPullV];
#pragma unroll
      for (int u = 0; u < kPullV; ++u) {
        const int64_t g = g0 + u * 32 + lane;
        sec[u] = g >= x1;
        src[u] = g < E ? ld_stream(a.col + (sec[u] ? s1 + (g - x1) : s0 + (g - x0))) : 0xffffffffu;
      }
      typename Op::A xa = 0, xb = 0;
#pragma unroll
      for (int u = 0; u < kPullV; ++u) {
        my_proc += src[u] != 0xffffffffu;
        const typename Op::A y = src[u] != 0xffffffffu ? op.load(src[u]) : typename Op::A(0);
        if (sec[u]) xb += y;
        else xa += y;
      }
      xa = warp_sum(xa);
      xb = warp_sum(xb);
      if (lane == 0) {
        atomicAdd(hacc + o, xa);
        if (x1 < g0 + CH && x1 < E) atomicAdd(hacc + o + 1, xb);
      }
    }
    cta_flush(a, my_proc, ctl->round);
    return;
  }
  for (int64_t p0 = 0; p0 < passes; p0 += kU) {
    int o[kU];
    uint32_t src[kU];
    typename Op::A x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t p = p0 + u;
      const int64_t g = BLOCKED ? tid * passes + p : p * T + tid;
      o[u] = -1;
      src[u] = 0;
      if (p < passes && g < E) {
        o[u] = (int)owner_search(pre, nh, g);
        src[u] = ld_stream(a.col + a.hstart[o[u]] + (g - (o[u] ? pre[o[u] - 1] : 0)));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      x[u] = o[u] >= 0 ? op.load(src[u]) : typename Op::A(0);
      my_proc += o[u] >= 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        typename Op::A y = __shfl_up_sync(kFull, x[u], dd);
        int oo = __shfl_up_sync(kFull, o[u], dd);
        if (lane >= (uint32_t)dd && oo == o[u]) x[u] += y;
      }
      int onext = __shfl_down_sync(kFull, o[u], 1);
      bool last = (lane == 31) || onext != o[u];
      if (o[u] >= 0 && last) atomicAdd(hacc + o[u], x[u]);
    }
  }
  cta_flush(a, my_proc, ctl->round);
}

// tiled pr: per-block static bin counts {nhuge, huge_edges, nlarge, large_edges}
static __global__ void k_tile_store(Ctl *ctl, long long *meta) {
  if (threadIdx.x) return;
  meta[0] = ctl->nhuge, meta[1] = (long long)ctl->huge_edges;
  meta[2] = ctl->nlarge, meta[3] = (long long)ctl->large_edges;
  ctl->nhuge = ctl->nlarge = 0;
  ctl->huge_edges = ctl->large_edges = 0;
}
static __global__ void k_tile_select(Ctl *ctl, const long long *meta) {
  if (threadIdx.x || ctl->done) return;
  ctl->nhuge = (uint32_t)meta[0], ctl->huge_edges = (unsigned long long)meta[1];
  ctl->nlarge = (uint32_t)meta[2], ctl->large_edges = (unsigned long long)meta[3];
  ctl->large_head = ctl->chunk_head = 0;
}

// huge-row fold (single CTA; huge rows are few) — plus the pr round advance
struct PrStop {            // apps.py:163-171, 183-185 evaluated on the device
  const unsigned long long *gain_max_bits;  // max_v sum_{u->v} inv_outdeg[u]
  double damping, tol;
  int64_t ne;              // active edges per round (all of E)
  int64_t limit;           // min(max_rounds, stats capacity)
  int64_t max_rounds;
  cudaGraphConditionalHandle cond;
  int use_cond;
  int parts_nonempty;      // devices > 1: partitions with rows (each launches every round)
  // 0: single process (fold + stop); 1: rank-local half (fold huge rows, local
  // delta / comm_bcast into Ctl, no decision); 2: global half after the
  // all-reduce (stats + stop from the reduced Ctl fields and `dist`)
  int mode;
  const long long *dist;   // mode 2: DistPr counters summed over ranks
  const long long *bins;   // tiled pr: {nhuge, huge_edges, nlarge, large_edges} of the full CSC
};

template <class Op, bool PR>
__global__ void __launch_bounds__(1024) k_pull_finish(PullArgs a, Op op,
                                                      typename Op::A *hacc, PrStop stop) {
  __shared__ double redd[32];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  op.begin(round);
  const uint32_t nh = ctl->nhuge;
  if (stop.mode != 2) {
    for (uint32_t i = threadIdx.x; i < nh; i += 1024) {
      typename Op::A acc = hacc[i];
      hacc[i] = 0;
      uint32_t v = a.hugeq[i];
      if (op.finish(v, acc)) a.dying[atomicAdd(&ctl->ndying, 1u)] = v;
    }
  }
  if (!PR) return;
  __shared__ unsigned long long redb[32];
  if (a.mcount && stop.mode != 2) {
    unsigned long long b = block_sum(op.bcast, redb);
    if (threadIdx.x == 0 && b) atomicAdd(&ctl->comm_bcast, b);
  }
  double m = warp_max(op.dmax);
  if (lane_id() == 0) redd[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 32; ++w) m = redd[w] > m ? redd[w] : m;
    unsigned long long mb = (unsigned long long)__double_as_longlong(m);
    if (stop.mode == 1) {  // rank-local half: the all-reduce and mode 2 follow
      atomicMax(&ctl->delta_bits, mb);
      return;
    }
    unsigned long long old = stop.mode == 2 ? ctl->delta_bits : atomicMax(&ctl->delta_bits, mb);
    double delta = __longlong_as_double((long long)(old > mb ? old : mb));
    double worst = __dmul_rn(stop.damping, __longlong_as_double((long long)*stop.gain_max_bits));
    double eps_stop = stop.tol / (worst > 1.0 ? worst : 1.0);
    RoundStat &st = a.stats[round];
    st.frontier_size = a.nv;
    st.active_edges = stop.ne;
    const bool g2 = stop.mode == 2;  // dist = {twc, lb, nhuge, huge_edges, nlarge, large_edges}
    st.huge_count = g2 ? stop.dist[2] : stop.bins ? stop.bins[0] : nh;
    st.huge_edges = g2 ? stop.dist[3] : stop.bins ? stop.bins[1] : (long long)ctl->huge_edges;
    st.large_count = g2 ? stop.dist[4] : stop.bins ? stop.bins[2] : ctl->nlarge;
    st.large_edges = g2 ? stop.dist[5] : stop.bins ? stop.bins[3] : (long long)ctl->large_edges;
    st.updated = a.nv;
    st.comm_sent = 0;
    st.comm_broadcast = (long long)ctl->comm_bcast;
    st.launches_twc = stop.mode == 2 ? stop.dist[0] : a.cuts.D > 1 ? stop.parts_nonempty : 1;
    st.launches_lb = stop.mode == 2 ? stop.dist[1]
                     : a.cuts.D > 1  ? __popc(ctl->part_lb_mask)
                     : stop.bins     ? stop.bins[0] > 0
                                     : nh > 0;
    ctl->comm_bcast = 0;
    ctl->delta_bits = 0;
    ctl->large_head = 0;
    ctl->chunk_head = 0;
    ctl->round = round + 1;
    if (delta <= eps_stop) ctl->done = 1;  // apps.py:183-185
    else if ((int64_t)round + 1 >= stop.limit)
      ctl->error = (int64_t)round + 1 >= stop.max_rounds ? SG_ECONVERGE : SG_ENOMEM, ctl->done = 1;
    if (stop.use_cond) cudaGraphSetConditional(stop.cond, ctl->done ? 0u : 1u);
  }
}

}  // namespace sg
