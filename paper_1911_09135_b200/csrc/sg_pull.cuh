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
#include "sg_push.cuh"

namespace sg {

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
};

// pr: acc = sum aux[u]; new = (1-d) + d*acc (two roundings, as numpy); aux' = new*inv
struct PrOp {
  using A = double;
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
  __device__ __forceinline__ void begin(uint32_t round) {
    aux = (round & 1) ? aux1 : aux0;
    auxn = (round & 1) ? next1 : next0;
  }
  __device__ __forceinline__ A load(uint32_t u) const { return __ldg(aux + u); }
  __device__ __forceinline__ bool finish(uint32_t v, A acc) {
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
  const bool dense = !a.dynamic_bins || ctl->dense;
  const uint32_t n = dense ? a.nv : ctl->fsize;
  const uint32_t *list = (round & 1) ? a.q[1] : a.q[0];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  unsigned long long my_edges = 0, my_large = 0;
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarpsTB;
  for (uint64_t c = (uint64_t)blockIdx.x * kWarpsTB + warp; c * 32 < n; c += nwarps) {
    uint64_t i = c * 32 + lane;
    uint32_t v = 0;
    int64_t s = 0, deg = 0;
    const bool valid = i < n;
    if (valid) {
      v = dense ? (uint32_t)i : list[i];
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
    const bool mine = valid && !huge && !large;
    const uint32_t gd = mine ? (uint32_t)deg : 0u;
    const uint32_t incl = warp_incl_scan(gd);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - gd;
    typename Op::A acc = 0;
    for (uint32_t base = 0; base < total; base += 32 * kU) {
      int o[kU];
      uint32_t src[kU];
      typename Op::A x[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // kU adjacency loads in flight
        const uint32_t slot = base + u * 32 + lane;
        o[u] = warp_owner(incl, slot);
        const int64_t so = shfl64(s, o[u]);
        const uint32_t eo = __shfl_sync(kFull, excl, o[u]);
        src[u] = slot < total ? ld_stream(a.col + so + (slot - eo)) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)  // then kU value gathers in flight
        x[u] = src[u] != 0xffffffffu ? op.load(src[u]) : typename Op::A(0);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
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
}

// TWC CTA bin: one CTA per row (dynamic fetch), deterministic tree reduction
template <class Op>
__global__ void __launch_bounds__(kTB) k_pull_large(PullArgs a, Op op) {
  __shared__ typename Op::A red[32];
  __shared__ uint32_t item;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t n = ctl->nlarge;
  if (!n) return;
  op.begin(ctl->round);
  for (;;) {
    if (threadIdx.x == 0) item = atomicAdd(&ctl->large_head, 1u);
    __syncthreads();
    const uint32_t idx = item;
    __syncthreads();
    if (idx >= n) break;
    const uint32_t v = a.largeq[idx];
    const int64_t s = a.off[v], e = a.off[v + 1];
    typename Op::A x = 0;
    for (int64_t b = s + threadIdx.x; b < e; b += kTB * kU) {
      uint32_t src[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) src[u] = b + u * kTB < e ? ld_stream(a.col + b + u * kTB) : 0xffffffffu;
#pragma unroll
      for (int u = 0; u < kU; ++u) x += src[u] != 0xffffffffu ? op.load(src[u]) : typename Op::A(0);
    }
    x = block_sum(x, red);
    if (threadIdx.x == 0 && op.finish(v, x)) a.dying[atomicAdd(&ctl->ndying, 1u)] = v;
  }
  if (sizeof(typename Op::A) == 8 && threadIdx.x == 0 && op.dmax > 0)
    atomic_max_dbits(&ctl->delta_bits, op.dmax);
  if (threadIdx.x == 0 && op.bcast) atomicAdd(&ctl->comm_bcast, op.bcast);
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
    for (int u = 0; u < kU; ++u) x[u] = o[u] >= 0 ? op.load(src[u]) : typename Op::A(0);
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
  for (uint32_t i = threadIdx.x; i < nh; i += 1024) {
    typename Op::A acc = hacc[i];
    hacc[i] = 0;
    uint32_t v = a.hugeq[i];
    if (op.finish(v, acc)) a.dying[atomicAdd(&ctl->ndying, 1u)] = v;
  }
  if (!PR) return;
  __shared__ unsigned long long redb[32];
  if (a.mcount) {
    unsigned long long b = block_sum(op.bcast, redb);
    if (threadIdx.x == 0 && b) atomicAdd(&ctl->comm_bcast, b);
  }
  double m = warp_max(op.dmax);
  if (lane_id() == 0) redd[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 32; ++w) m = redd[w] > m ? redd[w] : m;
    unsigned long long mb = (unsigned long long)__double_as_longlong(m);
    unsigned long long old = atomicMax(&ctl->delta_bits, mb);
    double delta = __longlong_as_double((long long)(old > mb ? old : mb));
    double worst = __dmul_rn(stop.damping, __longlong_as_double((long long)*stop.gain_max_bits));
    double eps_stop = stop.tol / (worst > 1.0 ? worst : 1.0);
    RoundStat &st = a.stats[round];
    st.frontier_size = a.nv;
    st.active_edges = stop.ne;
    st.huge_count = nh;
    st.huge_edges = (long long)ctl->huge_edges;
    st.large_count = ctl->nlarge;
    st.large_edges = (long long)ctl->large_edges;
    st.updated = a.nv;
    st.comm_sent = 0;
    st.comm_broadcast = (long long)ctl->comm_bcast;
    st.launches_twc = a.cuts.D > 1 ? stop.parts_nonempty : 1;
    st.launches_lb = a.cuts.D > 1 ? __popc(ctl->part_lb_mask) : nh > 0;
    ctl->comm_bcast = 0;
    ctl->delta_bits = 0;
    ctl->large_head = 0;
    ctl->round = round + 1;
    if (delta <= eps_stop) ctl->done = 1;  // apps.py:183-185
    else if ((int64_t)round + 1 >= stop.limit)
      ctl->error = (int64_t)round + 1 >= stop.max_rounds ? SG_ECONVERGE : SG_ENOMEM, ctl->done = 1;
    if (stop.use_cond) cudaGraphSetConditional(stop.cond, ctl->done ? 0u : 1u);
  }
}

}  // namespace sg
