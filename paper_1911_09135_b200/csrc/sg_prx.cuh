// sg_prx.cuh — pr pull rounds with the reference's exact summation order.
//
// Reference: OP_PULL_ADD out[row] += aux[col[e]] applied by np.add.at in array
// order (_kernels_py.py:73-75), i.e. every row is summed left to right in CSC
// order from 0.0; new = (1-d) + d*acc (apps.py:180); stop on max|new-old| <=
// eps_stop with eps_stop from np.bincount sums in the same order (apps.py:163-
// 171).  Floating-point addition is not associative, so a tree or atomic sum
// changes the labels in the last bits and, near eps_stop, the round the stop
// test fires in.  Here every sum is the reference's sequential one, bit for bit:
//
//  * short rows (deg < hs, ExactLayout SELL slices): one lane per row adds its
//    row's values in order -- fully coalesced adjacency loads, no shuffles.
//  * long rows: 256-edge chunks.  While a running sum s stays inside one binade
//    [2^e, 2^(e+1)), every sequential step fl(s + x) lands on the grid of
//    u = 2^(e-52), so fl(s + x) = s + r*u with r = x/u rounded to nearest
//    (ties: to the even significand, which depends on s).  A chunk's
//    sequential sum is therefore s + (sum of r)*u, computed exactly in int64 by
//    a warp reduction -- valid when no value is a tie and the sum does not
//    leave the binade (N0 + R < 2^53, N0 = s/u; the r are >= 0, so every
//    partial sum is then inside).  Otherwise the chunk is added serially
//    (binade crossings: ~log2 of the row length per row; ties: a value exactly
//    on a half-ulp).
//  * ALB huge rows (deg >= threshold): the chunks are spread over all warps,
//    each computing its R against a guessed binade (the one the row's sum had
//    at that chunk in the previous pass); one walker warp per row then chains
//    the chunks in order, O(1) per chunk when the guess holds, and redoes a
//    chunk exactly when it does not.  Other long rows ("self" rows, and every
//    long row of a TWC-only run) are walked chunk by chunk by one warp.
#pragma once
#include <climits>
#include <cstdlib>

#include "sg_pull.cuh"

namespace sg {
namespace {  // per translation unit, like sg_runtime.cuh

constexpr int kXV = 8;              // values per lane per 256-edge chunk
constexpr int kXChunk = 32 * kXV;   // edges per chunk
constexpr int kNoGuess = INT_MIN;

// rows shorter than exact_hs() go to the SELL slices, longer ones to 256-edge
// chunks (swept 128..8192 on rmat24: profiles/r2d, r2f); SG_EXACT_HS overrides
inline int64_t exact_hs() {
  static const int64_t hs = [] {
    const char *e = std::getenv("SG_EXACT_HS");
    const int64_t x = e ? std::atoll(e) : 2048;
    return std::max<int64_t>(2, std::min<int64_t>(x, 8192));
  }();
  return hs;
}

__global__ void k_copy_f64(const double *__restrict__ a, int64_t n, double *__restrict__ b) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) b[i] = a[i];
}

struct PrxArgs {
  const int64_t *off;
  const uint32_t *col;
  // ExactLayout of this view
  const uint32_t *srow;
  const uint8_t *sflag;
  const int64_t *soff;
  const uint32_t *scol;
  uint32_t nslices;
  const uint32_t *gfirst;     // [ngroups + 1] slice groups (dynamic-fetch units)
  uint32_t ngroups;
  const uint32_t *big;
  const uint8_t *bflag;
  uint32_t nsplit, nself;     // big[0, nsplit): ALB huge rows, [nsplit, nsplit + nself): walked
  const uint32_t *ck_first;   // [nsplit + 1] first chunk of each huge row
  const uint32_t *ck_row;     // [nchunks] huge row of each chunk
  uint32_t nchunks;
  long long *ck_T;            // chunk sums in units of the guessed ulp
  uint32_t *ck_meta;          // stamp << 2 | tie << 1 | guess valid
  int *ck_guess;              // exponent of the row's sum at the chunk's start (last pass)
  uint32_t *head;             // this pass's dynamic fetch counter
  Ctl *ctl;
  double *carry;              // tiled csc: partial row sums between source blocks
  int gain;                   // 1: eps_stop gain pass (aux = inv_outdeg, fold = max)
  unsigned long long *gain_bits;
  unsigned long long *cta_edges;
  uint32_t cta_g, cta_rounds;
};

struct PrFold {
  const double *aux0, *aux1;
  double *next0, *next1;
  double *rank;
  const double *inv;
  double d, omd;
  const uint32_t *mcount;  // devices > 1 (simulated partitions): comm_broadcast
  const double *aux = nullptr;
  double *auxn = nullptr;
  double dmax = 0.0;
  unsigned long long bcast = 0;
  __device__ __forceinline__ void begin(uint32_t round, int gain) {
    aux = gain ? inv : (round & 1) ? aux1 : aux0;
    auxn = (round & 1) ? next1 : next0;
  }
  __device__ __forceinline__ void fold(uint32_t v, double acc, int gain) {
    if (gain) {  // gain[v] = sum_{u->v} inv_outdeg[u] (apps.py:166-168)
      dmax = acc > dmax ? acc : dmax;
      return;
    }
    const double nw = __dadd_rn(omd, __dmul_rn(d, acc));  // apps.py:180, two roundings
    const double old = rank[v];
    const double dl = fabs(__dsub_rn(nw, old));
    dmax = dl > dmax ? dl : dmax;
    if (mcount && nw != old) bcast += mcount[v];  // engine.py:232-234
    rank[v] = nw;
    auxn[v] = __dmul_rn(nw, inv[v]);  // apps.py:176-177
  }
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// unbiased exponent of a positive normal double (s in [2^e, 2^(e+1)))
__device__ __forceinline__ int dexp(double s) {
  return (int)((__double_as_longlong(s) >> 52) & 0x7ff) - 1023;
}
__device__ __forceinline__ double pow2(int k) {  // 2^k, |k| < 1023
  return __longlong_as_double((long long)(1023 + k) << 52);
}
constexpr long long kTwo53 = 1ll << 53;
__device__ __forceinline__ bool exp_ok(int e) { return e > -900 && e < 900; }

// this lane's values rounded to the grid 2^(e-52) (units), and whether one is a tie
__device__ __forceinline__ long long grid_units(const double (&x)[kXV], int e, int &tie) {
  const double iu = pow2(52 - e);
  long long r = 0;
#pragma unroll
  for (int u = 0; u < kXV; ++u) {
    const double q = x[u] * iu;  // exact: a power-of-two scaling
    if (q >= 9007199254740992.0) {
      r += kTwo53;  // >= one binade: the chunk leaves it
    } else {
      const double m = floor(q), f = q - m;  // both exact
      r += (long long)m + (f > 0.5 ? 1 : 0);
      tie |= f == 0.5;
    }
  }
  return r;
}

// s := the sequential sum s + x_0 + x_1 + ... over the chunk's 256 values in
// slot order (slot = u * 32 + lane); s is warp-uniform
__device__ __forceinline__ double ex_step(double s, const double (&x)[kXV]) {
  if (s > 0.0) {
    const int e = dexp(s);
    if (exp_ok(e)) {
      int tie = 0;
      long long R = warp_sum(grid_units(x, e, tie));
      const long long N0 = (long long)(s * pow2(52 - e));
      if (!__any_sync(kFull, tie) && N0 + R < kTwo53) return (double)(N0 + R) * pow2(e - 52);
    }
  }
#pragma unroll
  for (int u = 0; u < kXV; ++u) {
#pragma unroll 8
    for (int l = 0; l < 32; ++l) s = __dadd_rn(s, __shfl_sync(kFull, x[u], l));
  }
  return s;
}

__device__ __forceinline__ void gather_src(const uint32_t *col, int64_t n, uint32_t (&src)[kXV]) {
#pragma unroll
  for (int u = 0; u < kXV; ++u) {
    const int64_t j = u * 32 + lane_id();
    src[u] = j < n ? ld_stream(col + j) : ExactLayout::kEmpty;
  }
}
__device__ __forceinline__ void gather_val(const double *aux, const uint32_t (&src)[kXV],
                                           double (&x)[kXV]) {
#pragma unroll
  for (int u = 0; u < kXV; ++u) x[u] = src[u] != ExactLayout::kEmpty ? __ldg(aux + src[u]) : 0.0;
}

__device__ __forceinline__ double row_start(const PrxArgs &a, uint32_t v, uint8_t f) {
  return (f & ExactLayout::kFirst) ? 0.0 : a.carry[v];
}
__device__ __forceinline__ void row_end(const PrxArgs &a, PrFold &op, uint32_t v, uint8_t f,
                                        double acc) {
  if (f & ExactLayout::kLast) op.fold(v, acc, a.gain);
  else a.carry[v] = acc;
}

// one warp walks row v's chunks [k0, nk) in order from s; software-pipelined:
// chunk k is added while the values of k + 1 and the columns of k + 2 load
__device__ __forceinline__ double walk_chunks(const PrxArgs &a, const PrFold &op, int64_t s0,
                                              int64_t d, int64_t k0, int64_t nk, double s,
                                              unsigned long long &proc) {
  if (k0 >= nk) return s;
  uint32_t sb[kXV], sc[kXV] = {};
  double xa[kXV], xb[kXV];
  gather_src(a.col + s0 + k0 * kXChunk, d - k0 * kXChunk, sb);
  gather_val(op.aux, sb, xa);
  if (k0 + 1 < nk) gather_src(a.col + s0 + (k0 + 1) * kXChunk, d - (k0 + 1) * kXChunk, sb);
  for (int64_t k = k0; k < nk; ++k) {
    if (k + 1 < nk) gather_val(op.aux, sb, xb);
    if (k + 2 < nk) gather_src(a.col + s0 + (k + 2) * kXChunk, d - (k + 2) * kXChunk, sc);
    s = ex_step(s, xa);
#pragma unroll
    for (int u = 0; u < kXV; ++u) xa[u] = xb[u], sb[u] = sc[u];
  }
  if (lane_id() == 0) proc += (unsigned long long)(d - k0 * kXChunk);
  return s;
}

// ALB huge row: chunk t against its guessed binade
__device__ __forceinline__ void split_chunk(const PrxArgs &a, const PrFold &op, uint32_t t,
                                            uint32_t stamp, unsigned long long &proc) {
  const uint32_t i = a.ck_row[t], v = a.big[i];
  const int64_t s0 = a.off[v], d = a.off[v + 1] - s0;
  const int64_t k = (int64_t)(t - a.ck_first[i]);
  uint32_t src[kXV];
  double x[kXV];
  gather_src(a.col + s0 + k * kXChunk, d - k * kXChunk, src);
  gather_val(op.aux, src, x);
  const int g = __ldcg(a.ck_guess + t);
  const bool valid = g != kNoGuess && exp_ok(g);
  int tie = 0;
  long long R = valid ? warp_sum(grid_units(x, g, tie)) : 0;
  tie = __any_sync(kFull, tie);
  if (lane_id() == 0) {
    a.ck_T[t] = R;
    st_release_u32(a.ck_meta + t, (stamp << 2) | (tie ? 2u : 0u) | (valid ? 1u : 0u));
    const int64_t n = d - k * kXChunk;
    proc += (unsigned long long)(n < kXChunk ? n : kXChunk);
  }
}

// ALB huge row i: chain its chunks
__device__ __forceinline__ void split_walk(const PrxArgs &a, PrFold &op, uint32_t i,
                                           uint32_t stamp, unsigned long long &proc) {
  const uint32_t v = a.big[i];
  const uint8_t f = a.bflag[i];
  const uint32_t c0 = a.ck_first[i], c1 = a.ck_first[i + 1];
  const int64_t s0 = a.off[v], d = a.off[v + 1] - s0;
  double s = row_start(a, v, f);
  const uint32_t lane = lane_id();
  // lane l holds chunk base + l of the current batch; the next batch's
  // results are loaded while this one is folded (a dependent load per batch
  // was the walker's critical path on heavy-skew hub rows)
  auto fetch = [&](uint32_t b, long long &T, uint32_t &meta, int &g) {
    const uint32_t j = b + lane;
    T = 0, meta = 0, g = kNoGuess;
    if (j < c1) {
      meta = ld_acquire_u32(a.ck_meta + j);  // then T / g: ordered after it
      T = __ldcg(a.ck_T + j);
      g = __ldcg(a.ck_guess + j);
    }
  };
  long long T;
  uint32_t meta;
  int g;
  fetch(c0, T, meta, g);
  for (uint32_t base = c0; base < c1; base += 32) {
    const uint32_t j = base + lane;
    if (j < c1)
      while ((meta >> 2) != stamp) {  // not this pass's result yet: wait, reload
        __nanosleep(100);
        meta = ld_acquire_u32(a.ck_meta + j);
        T = __ldcg(a.ck_T + j);
        g = __ldcg(a.ck_guess + j);
      }
    long long Tn = 0;
    uint32_t mn = 0;
    int gn = kNoGuess;
    if (base + 32 < c1) fetch(base + 32, Tn, mn, gn);
    const uint32_t m = min(32u, c1 - base);
    uint32_t tt = 0;
    while (tt < m) {
      const int es = s > 0.0 ? dexp(s) : kNoGuess;
      // bulk: the longest run of chunks tt.. whose sums were formed on the
      // current binade's grid (no tie, guess == es) -- inside one binade the
      // sequential sum is the integer sum N0 + T_tt + T_tt+1 + ..., so the
      // run is one warp prefix sum instead of one dependent step per chunk
      const bool mine = lane >= tt && lane < m;
      const bool ok = mine && s > 0.0 && exp_ok(es) && (meta & 1u) && !(meta & 2u) && g == es;
      const uint32_t bad = __ballot_sync(kFull, mine && !ok);
      uint32_t end = bad ? (uint32_t)(__ffs(bad) - 1) : m;
      if (end > tt) {
        const long long N0 = (long long)(s * pow2(52 - es));
        const long long pre = warp_incl_scan(lane >= tt && lane < end ? T : 0ll);
        // ... and stays inside the binade (the T are >= 0: prefixes only grow)
        const uint32_t over = __ballot_sync(kFull, lane >= tt && lane < end && N0 + pre >= kTwo53);
        if (over) end = (uint32_t)(__ffs(over) - 1);
        if (end > tt) {
          if (lane >= tt && lane < end) a.ck_guess[j] = es;  // the next pass guesses this binade
          s = (double)(N0 + __shfl_sync(kFull, pre, end - 1)) * pow2(es - 52);
          tt = end;
          continue;
        }
      }
      // chunk tt alone: its own sum if it fits, else redone exactly from s
      const long long Tt = __shfl_sync(kFull, T, tt);
      const uint32_t mt = __shfl_sync(kFull, meta, tt);
      const int gt = __shfl_sync(kFull, g, tt);
      if (lane == tt) a.ck_guess[j] = es;
      bool done = false;
      if (s > 0.0 && (mt & 1u) && !(mt & 2u) && es == gt && exp_ok(es)) {
        const long long N0 = (long long)(s * pow2(52 - es));
        if (N0 + Tt < kTwo53) {
          s = (double)(N0 + Tt) * pow2(es - 52);
          done = true;
        }
      }
      if (!done) {  // redo the chunk exactly from s
        const int64_t k = (int64_t)(base + tt - c0);
        uint32_t src[kXV];
        double x[kXV];
        gather_src(a.col + s0 + k * kXChunk, d - k * kXChunk, src);
        gather_val(op.aux, src, x);
        s = ex_step(s, x);
      }
      ++tt;
    }
    T = Tn, meta = mn, g = gn;
  }
  if (lane == 0) row_end(a, op, v, f, s);
  (void)proc;
}

// one SELL slice: lane l sums row srow[32 s + l] in order
__device__ __forceinline__ void sell_slice(const PrxArgs &a, PrFold &op, uint32_t s,
                                           unsigned long long &proc) {
  const uint32_t lane = lane_id();
  const int64_t o = a.soff[s], len = (a.soff[s + 1] - o) >> 5;
  const uint32_t v = a.srow[(size_t)s * 32 + lane];
  const uint8_t f = a.sflag[(size_t)s * 32 + lane];
  double acc = v != ExactLayout::kEmpty ? row_start(a, v, f) : 0.0;
  const uint32_t *c = a.scol + o + lane;
  constexpr int U = 8;
  uint32_t src[U], srcn[U];
  unsigned long long n = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) src[u] = u < len ? ld_stream(c + 32 * u) : ExactLayout::kEmpty;
  for (int64_t j = 0; j < len; j += U) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      srcn[u] = j + U + u < len ? ld_stream(c + 32 * (j + U + u)) : ExactLayout::kEmpty;
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = src[u] != ExactLayout::kEmpty ? __ldg(op.aux + src[u]) : 0.0;
      n += src[u] != ExactLayout::kEmpty;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, x[u]);  // padding adds 0.0: exact
#pragma unroll
    for (int u = 0; u < U; ++u) src[u] = srcn[u];
  }
  proc += n;
  if (v != ExactLayout::kEmpty) row_end(a, op, v, f, acc);
}

#ifndef SG_PRX_SELL_MINB
#define SG_PRX_SELL_MINB 4  // the SELL-only pass (register cap 64; 6 CTAs / 40 regs measured -3 %)
#endif
#ifndef SG_PRX_MINB
#define SG_PRX_MINB 1  // min resident CTAs per SM (register cap) for k_prx
#endif
// PART 0: every ticket (huge-row chunks, walkers, long rows, SELL groups);
// PART 1: the long rows only; PART 2: the SELL groups only.  The single-device
// pr splits a pass into PART 1 + PART 2: the SELL code alone needs a third of
// the registers, so its launch keeps ~3x the warps in flight (the short rows'
// gathers are latency-bound: ncu on uniform rmat25, 107 registers = 2 CTAs/SM)
template <int PART>
__global__ void __launch_bounds__(kTB, PART == 2 ? SG_PRX_SELL_MINB : SG_PRX_MINB)
    k_prx(PrxArgs a, PrFold op) {
  __shared__ double redd[kWarpsTB];
  __shared__ unsigned long long redb[kWarpsTB];
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  op.begin(round, a.gain);
  const uint32_t stamp = a.gain ? 1u : round + 2u;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned long long proc = 0;
  const uint32_t n1 = a.nchunks, n2 = n1 + a.nsplit, n3 = n2 + a.nself;
  const uint32_t ntick = PART == 2 ? a.ngroups : n3 + (PART == 1 ? 0u : a.ngroups);
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.head, 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= ntick) break;
    if (PART == 2) {
      const uint32_t g0 = a.gfirst[t], g1 = a.gfirst[t + 1];
      for (uint32_t s = g0; s < g1; ++s) sell_slice(a, op, s, proc);
    } else if (t < n1) {
      split_chunk(a, op, t, stamp, proc);
    } else if (t < n2) {
      split_walk(a, op, t - n1, stamp, proc);
    } else if (t < n3) {
      const uint32_t i = a.nsplit + (t - n2), v = a.big[i];
      const uint8_t f = a.bflag[i];
      const int64_t s0 = a.off[v], d = a.off[v + 1] - s0;
      const double s = walk_chunks(a, op, s0, d, 0, (d + kXChunk - 1) / kXChunk,
                                   row_start(a, v, f), proc);
      if (lane == 0) row_end(a, op, v, f, s);
    } else {
      const uint32_t g0 = a.gfirst[t - n3], g1 = a.gfirst[t - n3 + 1];
      for (uint32_t s = g0; s < g1; ++s) sell_slice(a, op, s, proc);
    }
  }
  const double m = warp_max(op.dmax);
  const unsigned long long b = warp_sum(op.bcast);
  if (lane == 0) redd[warp] = m, redb[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = redd[0];
    unsigned long long bb = redb[0];
    for (int w = 1; w < kWarpsTB; ++w) mm = redd[w] > mm ? redd[w] : mm, bb += redb[w];
    if (mm > 0) atomic_max_dbits(a.gain ? a.gain_bits : &ctl->delta_bits, mm);
    if (bb) atomicAdd(&ctl->comm_bcast, bb);
  }
  const unsigned long long pc = warp_sum(proc);
  if (a.cta_edges && lane == 0 && pc && round < a.cta_rounds && !a.gain)
    atomicAdd(a.cta_edges + (size_t)round * a.cta_g + (sm_id() % a.cta_g), pc);
}


// first pass over a view (no previous binades): guesses from an approximate
// prefix of the chunk sums of every huge row (any order: only the exponent matters)
__global__ void __launch_bounds__(kTB) k_prx_guess_sums(PrxArgs a, const double *aux) {
  const uint32_t warps = (gridDim.x * kTB) >> 5;
  for (uint32_t t = (blockIdx.x * kTB + threadIdx.x) >> 5; t < a.nchunks; t += warps) {
    const uint32_t i = a.ck_row[t], v = a.big[i];
    const int64_t s0 = a.off[v], d = a.off[v + 1] - s0;
    const int64_t k = (int64_t)(t - a.ck_first[i]);
    uint32_t src[kXV];
    double x[kXV];
    gather_src(a.col + s0 + k * kXChunk, d - k * kXChunk, src);
    gather_val(aux, src, x);
    double y = 0;
#pragma unroll
    for (int u = 0; u < kXV; ++u) y += x[u];
    y = warp_sum(y);
    if (lane_id() == 0) a.ck_T[t] = __double_as_longlong(y);
  }
}
__global__ void __launch_bounds__(kTB) k_prx_guess_scan(PrxArgs a) {
  const uint32_t warps = (gridDim.x * kTB) >> 5;
  for (uint32_t i = (blockIdx.x * kTB + threadIdx.x) >> 5; i < a.nsplit; i += warps) {
    const uint32_t v = a.big[i];
    double run = (a.bflag[i] & ExactLayout::kFirst) ? 0.0 : a.carry[v];
    for (uint32_t base = a.ck_first[i]; base < a.ck_first[i + 1]; base += 32) {
      const uint32_t j = base + lane_id();
      const double y = j < a.ck_first[i + 1] ? __longlong_as_double(a.ck_T[j]) : 0.0;
      double incl = y;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const double z = __shfl_up_sync(kFull, incl, dd);
        if (lane_id() >= (uint32_t)dd) incl += z;
      }
      const double before = run + (incl - y);
      if (j < a.ck_first[i + 1]) a.ck_guess[j] = before > 0.0 ? dexp(before) : kNoGuess;
      run += __shfl_sync(kFull, incl, 31);
    }
  }
}

// chunk table of the huge rows: first chunk per row (exclusive scan of
// ceil(deg / 256)) and the row of every chunk; one CTA (huge rows are few)
__global__ void __launch_bounds__(1024) k_prx_chunks(const int64_t *off, const uint32_t *big,
                                                     uint32_t nsplit, uint32_t *ck_first,
                                                     uint32_t *ck_row) {
  __shared__ uint32_t red[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < nsplit; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    uint32_t c = 0;
    if (i < nsplit) {
      const uint32_t v = big[i];
      c = (uint32_t)((off[v + 1] - off[v] + kXChunk - 1) / kXChunk);
    }
    const uint32_t x = warp_incl_scan(c);
    if (lane_id() == 31) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) red[threadIdx.x] = warp_incl_scan(red[threadIdx.x]);
    __syncthreads();
    const uint32_t excl = carry + ((threadIdx.x >> 5) ? red[(threadIdx.x >> 5) - 1] : 0) + x - c;
    if (i < nsplit) {
      ck_first[i] = excl;
      for (uint32_t k = 0; k < c; ++k) ck_row[excl + k] = i;
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + c;
    __syncthreads();
  }
  if (threadIdx.x == 0) ck_first[nsplit] = carry;
}

// end of a pr round: stop test (apps.py:181-186) on the device, round log, reset
__global__ void k_prx_finish(Ctl *ctl, RoundStat *stats, uint32_t nv, PrStop stop, int D,
                             uint32_t *heads, int nheads) {
  if (threadIdx.x) return;
  if (ctl->done) {
    if (stop.use_cond) cudaGraphSetConditional(stop.cond, 0u);
    return;
  }
  const uint32_t round = ctl->round;
  const double delta = __longlong_as_double((long long)ctl->delta_bits);
  const double worst = __dmul_rn(stop.damping, __longlong_as_double((long long)*stop.gain_max_bits));
  const double eps_stop = stop.tol / (worst > 1.0 ? worst : 1.0);
  RoundStat &st = stats[round];
  st.frontier_size = nv;
  st.active_edges = stop.ne;
  st.huge_count = stop.bins[0];
  st.huge_edges = stop.bins[1];
  st.large_count = stop.bins[2];
  st.large_edges = stop.bins[3];
  st.updated = nv;
  st.comm_sent = 0;
  st.comm_broadcast = (long long)ctl->comm_bcast;
  st.launches_twc = D > 1 ? stop.parts_nonempty : 1;
  st.launches_lb = D > 1 ? __popc(ctl->part_lb_mask) : stop.bins[0] > 0;
  ctl->comm_bcast = 0;
  ctl->delta_bits = 0;
  for (int h = 0; h < nheads; ++h) heads[h] = 0;
  ctl->round = round + 1;
  if (delta <= eps_stop) ctl->done = 1;  // apps.py:183-185
  else if ((int64_t)round + 1 >= stop.limit)
    ctl->error = (int64_t)round + 1 >= stop.max_rounds ? SG_ECONVERGE : SG_ENOMEM, ctl->done = 1;
  if (stop.use_cond) cudaGraphSetConditional(stop.cond, ctl->done ? 0u : 1u);
}

// host: the arguments of one k_prx pass over view `bv` with layout `L`.  Big
// rows of degree >= split_min are ALB huge rows (split; none when !huge_on);
// `alloc(bytes)` provides the pass's device buffers (owned by the caller).
template <class Alloc>
PrxArgs prx_args(const View &bv, const ExactLayout &L, int64_t split_min, bool huge_on, Ctl *ctl,
                 double *carry, unsigned long long *gmax, uint32_t *head, Alloc &&alloc) {
  PrxArgs x{};
  x.off = bv.off.p, x.col = bv.col.p;
  x.srow = L.srow.p, x.sflag = L.sflag.p, x.soff = L.soff.p, x.scol = L.scol.p;
  x.nslices = (uint32_t)L.nslices;
  x.gfirst = L.gfirst.p, x.ngroups = (uint32_t)L.ngroups;
  x.big = L.big.p, x.bflag = L.bflag.p;
  int64_t nsplit = 0, nchunks = 0;
  if (huge_on)
    for (int64_t dg : L.big_deg) {
      if (dg < split_min) break;
      ++nsplit;
      nchunks += (dg + kXChunk - 1) / kXChunk;
    }
  if (nchunks > 0xffffffffLL) throw Error(SG_ERANGE, "pr: too many huge-row chunks");
  x.nsplit = (uint32_t)nsplit, x.nself = (uint32_t)(L.nbig - nsplit);
  x.nchunks = (uint32_t)nchunks;
  auto n1 = [](int64_t n) { return (size_t)std::max<int64_t>(n, 1); };
  x.ck_first = (uint32_t *)alloc(sizeof(uint32_t) * n1(nsplit + 1));
  x.ck_row = (uint32_t *)alloc(sizeof(uint32_t) * n1(nchunks));
  x.ck_T = (long long *)alloc(sizeof(long long) * n1(nchunks));
  x.ck_meta = (uint32_t *)alloc(sizeof(uint32_t) * n1(nchunks));
  x.ck_guess = (int *)alloc(sizeof(int) * n1(nchunks));
  x.head = head;
  x.ctl = ctl;
  x.carry = carry;
  x.gain_bits = gmax;
  return x;
}

}  // namespace
}  // namespace sg
