// sg_peer.cu — the edge-cut BSP over NVLink peer memory (one rank per GPU).
//
// Reference: make_partition / sync_labels / the per-device loop of
// engine.py:64-113, 184-235.  This is the B200 transport of the multi-GPU
// path: instead of packing updates and handing them to a collective library,
// the round's own kernels write straight into the other ranks' HBM over
// NVLink / NVSwitch (CUDA IPC mappings of one symmetric region per rank):
//
//   * storage (Gluon's outgoing edge cut): a rank holds only its own rows
//     [c[r], c[r+1]) of the traversal view -- sg_graph_partition slices them
//     out of a full graph (the full graph can then be dropped), so the
//     edge bytes per GPU fall as 1/N;
//   * labels: every rank keeps a full-length label copy in its region; the
//     copy of a vertex it owns is the master, the copy of a vertex its rows
//     point at is a mirror (engine.py:77-84), the rest is never read;
//   * push round (bfs / sssp / cc): the ALB round (sg_bm.cuh kernels, local
//     frontier = owned changed vertices) lowers local copies and sets bits of
//     the next-frontier bitmap (red.min / red.or); then
//       reduce   — every marked MIRROR: red.min of the local value into the
//                  owner's label and red.or into the owner's bitmap, straight
//                  over NVLink (comm_sent = these marks, exactly the
//                  reference's `out_d != baseline` pairs, engine.py:105-109);
//                  its last block to finish runs the device-side cross-GPU
//                  barrier (one system fence, relaxed flag stores, acquire
//                  polls);
//       compact  — every owner turns its marked rows into the next local
//                  frontier (+ snapshot labels) and stores each changed
//                  label into the ranks that hold it as a mirror (its
//                  mirror mask: only updated mirrors travel,
//                  comm_broadcast = their count, engine.py:232-234); its
//                  last block publishes the rank's counter block into every
//                  peer's slot, runs the barrier and advances: every rank
//                  sums the slots (round log + the device-side quiescence
//                  test, all ranks decide alike);
//   * pr: owners fold their CSC rows with the exact-order pull (sg_prx.cuh)
//     and store the new aux of each row into its mirror holders; max |delta|
//     and the counters go through the slots, the stop test is the reference's;
//   * kcore: owners count, kill, mark the neighbours of the dying (remote
//     stores of the round stamp into the owners' mark arrays), barrier, then
//     store the deaths into the mirror holders and collect their stamped rows
//     that are still alive.
//
// The whole BSP loop of a rank is ONE CUDA-graph launch (WHILE node): no host
// round trip and no collective library inside the loop.  The barrier spins
// on the device with a 60 s timeout (a rank that never arrives fails the run
// loudly instead of hanging the GPU).  The same code runs with ranks as host
// threads on one GPU (peers = plain device pointers), which is how the
// single-GPU tests drive it.
#include <chrono>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "sg_distk.cuh"
#include "sg_prx.cuh"

namespace sg {
namespace {

// ----------------------------------------------------- symmetric region --
constexpr int kSlot = 16;  // longs per counter slot
struct Hdr {
  unsigned long long bar[kMaxParts];  // barrier epochs: slot q is stored by rank q
  unsigned long long epoch;           // barriers this rank has entered
  unsigned long long err;             // a barrier timed out
  unsigned long long pad[14];
  long long cnt[2][kMaxParts][kSlot]; // counter blocks by round parity: slot q stored by rank q
};

// Byte layout of every rank's region (identical on all ranks of a team):
// header, next-frontier bitmap (bfs: visited), mirror-holding bitmap (setup),
// bfs round-start visited bitmap, three 8 B/V slabs (push: labels; pr: aux0 /
// aux1 / rank; kcore: alive / mark).
struct Layout {
  int64_t nv = 0;
  size_t nw = 0;
  size_t o_nb = 0, o_held = 0, o_prev = 0, o_d[3] = {0, 0, 0}, bytes = 0;
  static Layout of(int64_t nv) {
    auto al = [](size_t x) { return (x + 511) & ~(size_t)511; };
    Layout L;
    L.nv = nv;
    L.nw = (size_t)((nv + 31) / 32) + 1;
    size_t o = al(sizeof(Hdr));
    L.o_nb = o, o = al(o + 4 * L.nw);
    L.o_held = o, o = al(o + 4 * L.nw);
    L.o_prev = o, o = al(o + 4 * L.nw);  // bfs: visited bits as of the round start
    const size_t slab = al(8 * (size_t)std::max<int64_t>(nv, 1));
    for (int i = 0; i < 3; ++i) L.o_d[i] = o, o += slab;
    L.bytes = o;
    return L;
  }
};

struct TeamDev {
  char *base[kMaxParts];
  int rank, world;
};
template <class T>
__device__ __forceinline__ T *at(const TeamDev &t, int q, size_t off) {
  return reinterpret_cast<T *>(t.base[q] + off);
}
__device__ __forceinline__ Hdr *hdr(const TeamDev &t, int q) {
  return reinterpret_cast<Hdr *>(t.base[q]);
}

__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_volatile(const long long *p) {
  return *(const volatile long long *)p;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// red.min into a peer's (or this rank's) label over NVLink
__device__ __forceinline__ void red_min_sys(uint32_t *p, uint32_t v) { atomicMin_system(p, v); }
__device__ __forceinline__ void red_min_sys(unsigned long long *p, unsigned long long v) {
  atomicMin_system(p, v);
}

constexpr unsigned long long kBarrierNs = 60ull * 1000 * 1000 * 1000;

// Cross-GPU barrier: publish this rank's epoch into every peer's slot
// (release, system scope, after a system fence for the writes of the
// preceding kernels), then wait until every peer's epoch reached it (acquire).
// Skipped once the run is done (all ranks decide `done` from the same sums).
// One system fence, then relaxed flag stores (fence + strong store is the
// release pattern): st.release.sys carries its own system fence, about 1.4 us
// each on B200 (scripts/micro/fence.cu), so a store per peer would cost
// world x 1.4 us per barrier.
__device__ bool team_barrier_dev(const TeamDev &t, Ctl *ctl, bool fence = true) {
  Hdr *me = hdr(t, t.rank);
  const unsigned long long e = me->epoch + 1;
  me->epoch = e;
  if (fence) __threadfence_system();  // else the caller fenced
  for (int q = 0; q < t.world; ++q) st_relaxed_sys(&hdr(t, q)->bar[t.rank], e);
  const unsigned long long t0 = globaltimer();
  for (int q = 0; q < t.world; ++q)
    while (ld_acquire_sys(&me->bar[q]) < e) {
      if (globaltimer() - t0 > kBarrierNs) {
        me->err = 1;
        if (ctl) ctl->error = SG_ECUDA, ctl->done = 1;
        return false;
      }
      __nanosleep(40);
    }
  return true;
}
__global__ void k_team_barrier(TeamDev t, Ctl *ctl) {
  if (threadIdx.x || blockIdx.x) return;
  if (ctl && ctl->done) return;
  team_barrier_dev(t, ctl);
}

// grid of the ticketed exchange kernels: the tickets are same-address atomics
// (one per block), so the grid stays persistent-sized instead of one thread
// per word
inline int ticket_grid(int64_t n, int per_sm) {
  return std::min(grid_n(n), persistent_grid(per_sm));
}

// true in every thread of the grid's last block to finish (after all other
// blocks' writes, device scope); the ticket resets for the next launch.  The
// exchange kernels end with the barrier / the round's bookkeeping in that
// block instead of separate single-block launches.
__device__ __forceinline__ bool last_block(uint32_t *tick) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(tick, 1u) == gridDim.x - 1;
    if (last) *tick = 0u;
  }
  __syncthreads();
  return last;
}

// a run that went `done` outside an advance kernel (barrier timeout) leaves the loop
__global__ void k_loop_guard(const Ctl *ctl, Loop lp) {
  if (threadIdx.x || !lp.use_cond) return;
  if (ctl->done) cudaGraphSetConditional(lp.cond, 0u);
}

template <class L>
__global__ void k_copy_as(const uint32_t *src, int64_t n, L *dst) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    dst[i] = (L)src[i];
}

// bits of word w that are vertices in [lo, hi)
__device__ __forceinline__ uint32_t owned_bits(int64_t w, int64_t lo, int64_t hi) {
  const int64_t s = w * 32;
  const int64_t a = lo - s < 0 ? 0 : (lo - s > 32 ? 32 : lo - s);
  const int64_t b = hi - s < 0 ? 0 : (hi - s > 32 ? 32 : hi - s);
  if (b <= a) return 0u;
  return (uint32_t)((((1ull << b) - 1ull)) & ~((1ull << a) - 1ull));
}

// ------------------------------------------------------- mirror masks --
// ranks holding an owned vertex as a mirror: a bit per owned vertex (any
// holder) in front of the 4-byte rank mask, so the exchange kernels read the
// mask only for the vertices that have mirrors
struct Mirrors {
  const uint32_t *any;   // by global bitmap word: any[v / 32 - lo / 32] bit v % 32
  const uint32_t *mask;  // [hi - lo]
  int64_t lo;
  __device__ __forceinline__ uint32_t word(int64_t w) const { return any[w - (lo >> 5)]; }
  __device__ __forceinline__ uint32_t of(uint32_t v) const {
    return (word(v >> 5) >> (v & 31u)) & 1u ? mask[v - lo] : 0u;
  }
};

// setup 1: the vertices this rank's rows point at but does not own (its mirrors)
__global__ void k_px_held(const uint32_t *col, int64_t ne, int64_t lo, int64_t hi,
                          uint32_t *held) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += st) {
    const uint32_t v = col[e];
    if ((int64_t)v < lo || (int64_t)v >= hi) {
      const uint32_t bit = 1u << (v & 31u);
      if (!(held[v >> 5] & bit)) atomicOr(held + (v >> 5), bit);
    }
  }
}
// setup 2 (after a barrier): mask[v - lo] = ranks holding owned v as a mirror,
// mcount[v] = their number (engine.py:84 mirror_count)
__global__ void k_px_mask(TeamDev t, Layout lay, int64_t lo, int64_t hi, uint32_t *mask,
                          uint32_t *any, uint32_t *mcount) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < hi; v += st) {
    uint32_t m = 0;
    for (int q = 0; q < t.world; ++q) {
      if (q == t.rank) continue;
      const uint32_t w = *(const volatile uint32_t *)(at<uint32_t>(t, q, lay.o_held) + (v >> 5));
      if ((w >> (v & 31)) & 1u) m |= 1u << q;
    }
    mask[v - lo] = m;
    if (m) atomicOr(any + ((v >> 5) - (lo >> 5)), 1u << (v & 31));
    mcount[v] = (uint32_t)__popc(m);
  }
}

// ------------------------------------------------------- counter slots --
// this rank's counter block -> slot [rank] of every peer (parity of the round)
__global__ void k_px_publish(TeamDev t, const Ctl *ctl, const long long *acc, int n) {
  if (ctl && ctl->done) return;
  const int par = ctl ? (ctl->round & 1) : 0;
  for (int i = threadIdx.x; i < t.world * n; i += blockDim.x) {
    const int q = i / n, j = i % n;
    hdr(t, q)->cnt[par][t.rank][j] = acc[j];
  }
  __threadfence_system();
}
// after the barrier: acc[j] = sum (or max, bit j of max_mask) over the ranks' slots
__global__ void k_px_reduce_slots(TeamDev t, const Ctl *ctl, long long *acc, int n,
                                  uint32_t max_mask) {
  if (ctl && ctl->done) return;
  const int par = ctl ? (ctl->round & 1) : 0;
  const Hdr *me = hdr(t, t.rank);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    long long s = 0;
    for (int q = 0; q < t.world; ++q) {
      const long long x = ld_volatile(&me->cnt[par][q][j]);
      s = (max_mask >> j) & 1u ? (q == 0 || x > s ? x : s) : s + x;
    }
    acc[j] = s;
  }
}

// ----------------------------------------------------------- push apps --
// reduce: marked mirrors -> their owners (red.min label, red.or bitmap bit)
template <class L>
__global__ void __launch_bounds__(256) k_px_reduce(TeamDev t, Layout lay, Cuts cuts, Ctl *ctl,
                                                   long long *acc, uint32_t *tick) {
  __shared__ unsigned long long red[32];
  if (ctl->done) return;
  const int self = t.rank;
  uint32_t *nb = at<uint32_t>(t, self, lay.o_nb);
  const L *lab = at<L>(t, self, lay.o_d[0]);
  const int64_t lo = cuts.c[self], hi = cuts.c[self + 1];
  const int64_t nw = (lay.nv + 31) / 32, st = (int64_t)gridDim.x * blockDim.x;
  unsigned long long sent = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += st) {
    const uint32_t own = owned_bits(w, lo, hi);
    if (own == kFull) continue;
    uint32_t x = nb[w] & ~own;
    if (!x) continue;
    if (own) atomicAnd(nb + w, own);  // owners' peers may be setting the owned bits
    else nb[w] = 0u;
    sent += (unsigned long long)__popc(x);
    while (x) {
      const uint32_t v = (uint32_t)(w * 32) + (uint32_t)(__ffs(x) - 1);
      x &= x - 1;
      const int o = owner_of(cuts, v);
      red_min_sys(at<L>(t, o, lay.o_d[0]) + v, lab[v]);
      atomicOr_system(at<uint32_t>(t, o, lay.o_nb) + (v >> 5), 1u << (v & 31u));
    }
  }
  if (sent) __threadfence_system();  // only the threads that wrote to peers
  sent = block_sum(sent, red);
  if (threadIdx.x == 0 && sent) atomicAdd((unsigned long long *)&acc[6], sent);
  // every rank's reductions land before any owner compacts
  if (last_block(tick) && threadIdx.x == 0) team_barrier_dev(t, ctl);
}

// The round's tail, run by warp 0 of the compaction's last block: the
// counter block (k_dp_collect + the next-frontier size; sent and bcast were
// added by reduce / compact) goes into every peer's slot (lanes in parallel),
// the barrier, then every rank sums the same slots (lane j: slot j over the
// ranks), writes the same round log, decides quiescence identically and
// resets the round state; leaves the WHILE loop when the run is done for any
// reason (a barrier timeout included)
__device__ void push_round_tail(const PushArgs &a, const TeamDev &t, long long *acc,
                                const Loop &lp) {
  const uint32_t lane = lane_id();
  Ctl *ctl = a.ctl;
  if (lane == 0) {
    const long long fs = ctl->dense ? a.dense_n : (long long)ctl->fsize + ctl->fzero;
    acc[0] = fs;
    acc[1] = (long long)ctl->edges;
    acc[2] = a.sched >= 2 ? 0 : ctl->nhuge;
    acc[3] = a.sched >= 2 ? 0 : (long long)ctl->huge_edges;
    acc[4] = a.sched >= 2 ? 0 : ctl->nlarge;
    acc[5] = a.sched >= 2 ? 0 : (long long)ctl->large_edges;
    acc[8] = a.sched == 1 ? 0 : fs > 0;  // run_round only for a non-empty local frontier
    acc[9] = a.sched == 1 ? ctl->huge_edges > 0 : a.sched == 0 ? ctl->nhuge > 0 : 0;
    acc[10] = (long long)ctl->nsize + ctl->nzero;
  }
  __syncwarp();
  const int par = ctl->round & 1;
  for (int i = (int)lane; i < t.world * kDP; i += 32)
    hdr(t, i / kDP)->cnt[par][t.rank][i % kDP] = acc[i % kDP];
  __threadfence_system();
  __syncwarp();
  int ok = 1;
  if (lane == 0) ok = team_barrier_dev(t, ctl, false);
  ok = __shfl_sync(kFull, ok, 0);
  if (!ok) {
    if (lane == 0 && lp.use_cond) cudaGraphSetConditional(lp.cond, 0u);
    return;
  }
  const Hdr *me = hdr(t, t.rank);
  long long sum = 0;
  if (lane < (uint32_t)kDP)
    for (int q = 0; q < t.world; ++q) sum += ld_volatile(&me->cnt[par][q][lane]);
  long long x[kDP];
#pragma unroll
  for (int j = 0; j < kDP; ++j) x[j] = __shfl_sync(kFull, sum, j);
  if (lane) return;
  const uint32_t round = ctl->round;
  RoundStat &s = a.stats[round];
  s.frontier_size = x[0];
  s.active_edges = x[1];
  s.huge_count = x[2];
  s.huge_edges = x[3];
  s.large_count = x[4];
  s.large_edges = x[5];
  s.updated = x[10];
  s.comm_sent = x[6];
  s.comm_broadcast = x[7];
  s.launches_twc = x[8];
  s.launches_lb = x[9];
  ctl->fsize = ctl->nsize;
  ctl->fzero = ctl->nzero;
  ctl->nsize = ctl->nzero = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = ctl->chunk_head = 0;
  ctl->edges = ctl->huge_edges = ctl->large_edges = 0;
  ctl->dense = 0;
  ctl->round = round + 1;
  for (int j = 0; j < kDP; ++j) acc[j] = 0;
  loop_test(ctl, round, x[10] == 0, lp);
}
// a compaction launched after the run went done (barrier timeout) only leaves the loop
__device__ __forceinline__ bool done_exit(const Ctl *ctl, const Loop &lp) {
  if (!ctl->done) return false;
  if (blockIdx.x == 0 && threadIdx.x == 0 && lp.use_cond) cudaGraphSetConditional(lp.cond, 0u);
  return true;
}

// compact (after the barrier): owned marked rows -> next local frontier with
// their snapshot labels; each changed label is stored into its mirror holders.
// A warp takes 32 bitmap words and emits their set bits cooperatively (lane
// l emits slot l, l + 32, ...: a dense hot-set word block is 32 vertices per
// step, not 32 dependent steps of one lane)
template <class L>
__global__ void __launch_bounds__(256) k_px_compact(TeamDev t, Layout lay, Cuts cuts, PushArgs a,
                                                    Mirrors mm, uint32_t *q, L *snap,
                                                    long long *acc, uint32_t *tick, Loop lp,
                                                    uint32_t zlo) {
  __shared__ unsigned long long red[32];
  Ctl *ctl = a.ctl;
  if (done_exit(ctl, lp)) return;
  const int self = t.rank;
  uint32_t *nb = at<uint32_t>(t, self, lay.o_nb);
  const L *lab = at<L>(t, self, lay.o_d[0]);
  const int64_t lo = cuts.c[self], hi = cuts.c[self + 1];
  const uint32_t lane = lane_id();
  unsigned long long bc = 0;
  // the set bits of the warp's 32 words, lane l taking bit l, l + 32, ... in
  // word order, kE per lane in flight: queued (next frontier + snapshot) or,
  // for the edgeless tail [zlo, hi), only counted; both broadcast the label
  // to the vertex's mirror holders
  auto emit = [&](int64_t b, uint32_t x, bool queue) {
    const uint32_t n = (uint32_t)__popc(x);
    const uint32_t incl = warp_incl_scan(n);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (!total) return;
    uint32_t base = 0;
    if (queue && lane == 0) base = atomicAdd(&ctl->nsize, total);
    base = __shfl_sync(kFull, base, 0);
    const uint32_t excl = incl - n;
    constexpr int kE = 4;
    for (uint32_t k0 = 0; k0 < total; k0 += 32 * kE) {
      uint32_t v[kE], m[kE];
      L val[kE];
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const uint32_t slot = k0 + u * 32 + lane;
        const int o = warp_owner(incl, slot);
        const uint32_t xo = __shfl_sync(kFull, x, o);
        const uint32_t eo = __shfl_sync(kFull, excl, o);
        v[u] = slot < total ? (uint32_t)((b + o) * 32) + __fns(xo, 0, (int)(slot - eo) + 1) : 0u;
      }
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        m[u] = 0u;
        if (k0 + u * 32 + lane < total) {
          m[u] = mm.of(v[u]);
          if (queue || m[u]) val[u] = lab[v[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const uint32_t slot = k0 + u * 32 + lane;
        if (slot >= total) continue;
        if (queue) q[base + slot] = v[u], snap[base + slot] = val[u];
        bc += (unsigned long long)__popc(m[u]);
        while (m[u]) {
          const int r = __ffs(m[u]) - 1;
          m[u] &= m[u] - 1;
          at<L>(t, r, lay.o_d[0])[v[u]] = val[u];
        }
      }
    }
  };
  if (hi > lo) {
    const int64_t w0 = lo / 32, w1 = (hi - 1) / 32 + 1;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // warp-major over CTAs (as k_bm_compact): a dense run of frontier bits --
    // the relabeled hot set -- is spread over the SMs
    const int64_t gw = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    for (int64_t b = w0 + gw * 32; b < w1; b += warps * 32) {
      const int64_t w = b + lane;
      uint32_t x = 0, z = 0;
      if (w < w1) {
        x = nb[w] & owned_bits(w, lo, hi);
        if (x) nb[w] = 0u;  // the mirror bits of a boundary word were cleared by reduce
        z = x & owned_bits(w, zlo, hi);
      }
      emit(b, x & ~z, true);
      // the edgeless tail: counted; only its members with mirrors travel
      const uint32_t cz = __reduce_add_sync(kFull, (uint32_t)__popc(z));
      if (cz) {
        if (lane == 0) atomicAdd(&ctl->nzero, cz);
        const uint32_t za = z ? z & mm.word(w) : 0u;
        if (__any_sync(kFull, za)) emit(b, za, false);
      }
    }
  }
  if (bc) __threadfence_system();  // only the threads that wrote to peers
  bc = block_sum(bc, red);
  if (threadIdx.x == 0 && bc) atomicAdd((unsigned long long *)&acc[7], bc);
  if (last_block(tick) && threadIdx.x < 32) push_round_tail(a, t, acc, lp);
}

// ---- bfs: the visited-bitmap operator (BmBfs) over the peers.  vis (the nb
// slot) and prev (round-start vis) are full-length on every rank; a rank's
// mirror bits are exact at a round start (owners broadcast new vertices into
// both bitmaps of the mirror holders), so vis & ~prev on a mirror word is
// exactly what this rank discovered this round (`out_d != baseline`).
__global__ void __launch_bounds__(256) k_px_bfs_reduce(TeamDev t, Layout lay, Cuts cuts,
                                                       Ctl *ctl, long long *acc, uint32_t *tick) {
  __shared__ unsigned long long red[32];
  if (ctl->done) return;
  const int self = t.rank;
  const uint32_t *vis = at<uint32_t>(t, self, lay.o_nb);
  uint32_t *prev = at<uint32_t>(t, self, lay.o_prev);
  const int64_t lo = cuts.c[self], hi = cuts.c[self + 1];
  const int64_t nw = (lay.nv + 31) / 32, st = (int64_t)gridDim.x * blockDim.x;
  unsigned long long sent = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += st) {
    const uint32_t own = owned_bits(w, lo, hi);
    if (own == kFull) continue;
    const uint32_t x = vis[w] & ~prev[w] & ~own;
    if (!x) continue;
    if (own) atomicOr(prev + w, x);  // peers may set owned bits of a boundary word
    else prev[w] |= x;
    sent += (unsigned long long)__popc(x);
    uint32_t y = x;
    while (y) {
      const uint32_t v = (uint32_t)(w * 32) + (uint32_t)(__ffs(y) - 1);
      y &= y - 1;
      atomicOr_system(at<uint32_t>(t, owner_of(cuts, v), lay.o_nb) + (v >> 5), 1u << (v & 31u));
    }
  }
  if (sent) __threadfence_system();  // only the threads that wrote to peers
  sent = block_sum(sent, red);
  if (threadIdx.x == 0 && sent) atomicAdd((unsigned long long *)&acc[6], sent);
  // every rank's reductions land before any owner compacts
  if (last_block(tick) && threadIdx.x == 0) team_barrier_dev(t, ctl);
}

// owners: new owned bits -> next frontier, label round + 1; the vertex is
// marked visited in both bitmaps of its mirror holders
__global__ void __launch_bounds__(256) k_px_bfs_compact(TeamDev t, Layout lay, Cuts cuts,
                                                        PushArgs a, Mirrors mm,
                                                        uint32_t *q, long long *acc,
                                                        uint32_t *tick, Loop lp, uint32_t zlo) {
  __shared__ unsigned long long red[32];
  Ctl *ctl = a.ctl;
  if (done_exit(ctl, lp)) return;
  const int self = t.rank;
  const uint32_t *vis = at<uint32_t>(t, self, lay.o_nb);
  uint32_t *prev = at<uint32_t>(t, self, lay.o_prev);
  uint32_t *lab = at<uint32_t>(t, self, lay.o_d[0]);
  const uint32_t level = ctl->round + 1;
  const int64_t lo = cuts.c[self], hi = cuts.c[self + 1];
  const uint32_t lane = lane_id();
  unsigned long long bc = 0;
  // as k_px_compact: queued (next frontier) or, for the edgeless tail, only
  // counted; every new vertex gets its level and is marked in its mirror
  // holders' bitmaps
  auto emit = [&](int64_t b, uint32_t x, bool queue) {
    const uint32_t n = (uint32_t)__popc(x);
    const uint32_t incl = warp_incl_scan(n);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (!total) return;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(queue ? &ctl->nsize : &ctl->nzero, total);
    base = __shfl_sync(kFull, base, 0);
    const uint32_t excl = incl - n;
    constexpr int kE = 4;
    for (uint32_t k0 = 0; k0 < total; k0 += 32 * kE) {
      uint32_t v[kE], m[kE];
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const uint32_t slot = k0 + u * 32 + lane;
        const int o = warp_owner(incl, slot);
        const uint32_t xo = __shfl_sync(kFull, x, o);
        const uint32_t eo = __shfl_sync(kFull, excl, o);
        v[u] = slot < total ? (uint32_t)((b + o) * 32) + __fns(xo, 0, (int)(slot - eo) + 1) : 0u;
      }
#pragma unroll
      for (int u = 0; u < kE; ++u)
        if (k0 + u * 32 + lane < total) m[u] = mm.of(v[u]);
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const uint32_t slot = k0 + u * 32 + lane;
        if (slot >= total) continue;
        if (queue) q[base + slot] = v[u];
        lab[v[u]] = level;
        bc += (unsigned long long)__popc(m[u]);
        const uint32_t bit = 1u << (v[u] & 31u);
        while (m[u]) {
          const int r = __ffs(m[u]) - 1;
          m[u] &= m[u] - 1;
          atomicOr_system(at<uint32_t>(t, r, lay.o_nb) + (v[u] >> 5), bit);
          atomicOr_system(at<uint32_t>(t, r, lay.o_prev) + (v[u] >> 5), bit);
        }
      }
    }
  };
  if (hi > lo) {
    const int64_t w0 = lo / 32, w1 = (hi - 1) / 32 + 1;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t gw = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    for (int64_t b = w0 + gw * 32; b < w1; b += warps * 32) {
      const int64_t w = b + lane;
      uint32_t x = 0, z = 0;
      if (w < w1) {
        x = vis[w] & ~prev[w] & owned_bits(w, lo, hi);
        if (x) atomicOr(prev + w, x);
        z = x & owned_bits(w, zlo, hi);
      }
      emit(b, x & ~z, true);
      if (__any_sync(kFull, z)) emit(b, z, false);
    }
  }
  if (bc) __threadfence_system();  // only the threads that wrote to peers
  bc = block_sum(bc, red);
  if (threadIdx.x == 0 && bc) atomicAdd((unsigned long long *)&acc[7], bc);
  if (last_block(tick) && threadIdx.x < 32) push_round_tail(a, t, acc, lp);
}

// ------------------------------------------------------------- pr, kcore --
// every owned row's new value -> the ranks holding it as a mirror
template <class T>
__global__ void __launch_bounds__(256) k_px_rows(TeamDev t, size_t off0, size_t off1,
                                                 int parity_sel, const Ctl *ctl, int64_t lo,
                                                 int64_t hi, Mirrors mm) {
  if (ctl->done || hi <= lo) return;
  const size_t off = ((ctl->round & 1) == (uint32_t)parity_sel) ? off0 : off1;
  const T *src = at<T>(t, t.rank, off);
  // a warp takes 32 words of the any-mirror bitmap and walks only the words
  // with mirrors, one vertex per lane (no work for vertices without holders)
  const uint32_t lane = lane_id();
  const int64_t w0 = lo >> 5, w1 = ((hi - 1) >> 5) + 1;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool wrote = false;
  for (int64_t b = w0 + ((((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5)) * 32;
       b < w1; b += warps * 32) {
    const int64_t w = b + lane;
    const uint32_t word = w < w1 ? mm.word(w) & owned_bits(w, lo, hi) : 0u;
    uint32_t busy = __ballot_sync(kFull, word != 0u);
    while (busy) {
      const int j = __ffs(busy) - 1;
      busy &= busy - 1;
      const uint32_t wj = __shfl_sync(kFull, word, j);
      if (!((wj >> lane) & 1u)) continue;
      const uint32_t v = (uint32_t)((b + j) * 32) + lane;
      uint32_t m = mm.mask[v - lo];
      const T x = src[v];
      wrote = true;
      while (m) {
        const int r = __ffs(m) - 1;
        m &= m - 1;
        at<T>(t, r, off)[v] = x;
      }
    }
  }
  if (wrote) __threadfence_system();
}

// pr round tail in one warp (after the mirror rows): this rank's counters
// (k_dist_pr_collect's six, max |delta| bits, comm_broadcast) into every
// peer's slot, the barrier, then the sums (acc[6]: the max) back into acc and
// Ctl -- what collect / stage / publish / barrier / reduce_slots / unstage
// did in six launches
__global__ void k_px_pr_sync(TeamDev t, Ctl *ctl, int has_rows, long long *acc) {
  if (threadIdx.x >= 32 || ctl->done) return;
  const uint32_t lane = threadIdx.x;
  constexpr int n = 8;
  if (lane == 0) {
    acc[0] = has_rows;
    acc[1] = ctl->nhuge > 0;
    acc[2] = ctl->nhuge;
    acc[3] = (long long)ctl->huge_edges;
    acc[4] = ctl->nlarge;
    acc[5] = (long long)ctl->large_edges;
    acc[6] = (long long)ctl->delta_bits;  // a non-negative double: its bits order like it
    acc[7] = (long long)ctl->comm_bcast;
  }
  __syncwarp();
  const int par = ctl->round & 1;
  for (int i = (int)lane; i < t.world * n; i += 32) hdr(t, i / n)->cnt[par][t.rank][i % n] = acc[i % n];
  __threadfence_system();
  __syncwarp();
  int ok = 1;
  if (lane == 0) ok = team_barrier_dev(t, ctl, false);
  if (!__shfl_sync(kFull, ok, 0)) return;
  const Hdr *me = hdr(t, t.rank);
  if (lane < (uint32_t)n) {
    long long s = 0;
    for (int q = 0; q < t.world; ++q) {
      const long long x = ld_volatile(&me->cnt[par][q][lane]);
      s = lane == 6 ? (q == 0 || x > s ? x : s) : s + x;
    }
    acc[lane] = s;
  }
  __syncwarp();
  if (lane == 0) {
    ctl->delta_bits = (unsigned long long)acc[6];
    ctl->comm_bcast = (unsigned long long)acc[7];
  }
}


// kcore: this round's dying owned vertices -> alive = 0 at their mirror holders
__global__ void k_px_kill(TeamDev t, Layout lay, const Ctl *ctl, const uint32_t *dying,
                          Mirrors mm) {
  if (ctl->done) return;
  const uint32_t nd = ctl->ndying;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  bool wrote = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += st) {
    const uint32_t v = dying[i];
    uint32_t m = mm.of(v);
    wrote |= m != 0;
    while (m) {
      const int r = __ffs(m) - 1;
      m &= m - 1;
      at<uint8_t>(t, r, lay.o_d[0])[v] = 0;
    }
  }
  if (wrote) __threadfence_system();
}

// kcore mark phase over the peers: a neighbour of a dying vertex gets the
// round's stamp in its OWNER's mark array (a remote store when another rank
// owns it); after the barrier owners collect their stamped rows that are
// still alive (apps.py:226-231: alive = neighbours[values > 0] after the kill)
// -- the owner's alive flag is authoritative, so the mark phase needs no
// peer's deaths and the count phase never sees a death of its own round
struct OpMarkPeer {
  using L = uint32_t;
  static constexpr bool kCarry = false;
  const uint8_t *alive;  // this rank's copy (mirrors updated by k_px_kill)
  uint32_t *mark;        // this rank's mark array
  TeamDev t;
  size_t o_mark;
  Cuts cuts;
  uint32_t stamp = 0;
  __device__ __forceinline__ void begin(uint32_t round) { stamp = round + 1; }
  __device__ __forceinline__ L src_val(uint64_t, uint32_t) const { return 0; }
  __device__ __forceinline__ void sync_src(uint32_t, L) const {}
  __device__ __forceinline__ void relax(const PushArgs &a, const int64_t (&e)[kU],
                                        const bool (&ok)[kU], const L (&)[kU],
                                        uint32_t (&dst)[kU], bool (&act)[kU]) const {
    const long long lo = cuts.c[t.rank], hi = cuts.c[t.rank + 1];
    bool live[kU], own[kU];
    uint32_t cur[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) dst[u] = ok[u] ? ld_stream(a.col + e[u]) : 0u;
    // this rank's alive copy filters the vertices dead before this round (a
    // mirror's flag lags its owner by this round's deaths only: the owner
    // filters those when it collects)
#pragma unroll
    for (int u = 0; u < kU; ++u) live[u] = ok[u] && alive[dst[u]];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      own[u] = (long long)dst[u] >= lo && (long long)dst[u] < hi;
      cur[u] = live[u] && own[u] ? mark[dst[u]] : stamp;
    }
    // plain stores (nothing is enqueued here): the owner collects its stamped
    // rows after the barrier
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      act[u] = false;
      if (!live[u]) continue;
      if (own[u]) {
        if (cur[u] != stamp) mark[dst[u]] = stamp;
      } else {
        at<uint32_t>(t, owner_of(cuts, dst[u]), o_mark)[dst[u]] = stamp;
      }
    }
  }
};

// kcore: owned rows stamped this round and still alive -> next local frontier.
// A lane takes 4 vertices (one 16-byte mark load, one 4-byte alive load); one
// queue reservation per warp step
__global__ void k_px_kc_compact(const Ctl *ctl, const uint32_t *mark, const uint8_t *alive,
                                uint32_t lo, uint32_t hi, uint32_t *q0, uint32_t *q1,
                                uint32_t *nsize) {
  if (ctl->done) return;
  const uint32_t round = ctl->round, stamp = round + 1;
  uint32_t *q = (round & 1) ? q0 : q1;
  const uint64_t g0 = lo >> 2, g1 = ((uint64_t)hi + 3) >> 2;  // groups of 4 vertices
  const uint32_t lane = lane_id();
  const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < g1 - g0; b += st) {
    const uint64_t gi = g0 + b + threadIdx.x;
    const uint32_t v0 = (uint32_t)(gi * 4);
    uint32_t f = 0;
    if (gi < g1) {
      const uint4 m = reinterpret_cast<const uint4 *>(mark)[gi];
      const uint32_t al = reinterpret_cast<const uint32_t *>(alive)[gi];
      const uint32_t mv[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t v = v0 + k;
        if (v >= lo && v < hi && mv[k] == stamp && ((al >> (8 * k)) & 0xffu)) f |= 1u << k;
      }
    }
    const uint32_t c = (uint32_t)__popc(f);
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    if (!tot) continue;
    uint32_t base = 0;
    if (lane == 31) base = atomicAdd(nsize, tot);
    base = __shfl_sync(kFull, base, 31);
    uint32_t pos = base + incl - c;
    while (f) {
      const int k = __ffs(f) - 1;
      f &= f - 1;
      q[pos++] = v0 + (uint32_t)k;
    }
  }
}

// ---------------------------------------------------------- label gather --
// every rank's owned block -> this rank's full output (remote loads)
// (a relabeled partition: out[v] = the owner's value of inv[v]; the owner of
// v and of inv[v] is the same rank, the relabeling is block-local)
template <class T, class Conv>
__global__ void k_px_gather(TeamDev t, size_t off, Cuts cuts, int64_t nv, const uint32_t *inv,
                            double *out, Conv cv) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st) {
    const int o = owner_of(cuts, (uint32_t)v);
    const int64_t x = inv ? (int64_t)inv[v] : v;
    out[v] = cv(*(const volatile T *)(at<T>(t, o, off) + x));
  }
}
struct ConvU32 {
  __device__ double operator()(uint32_t x) const { return x == kInf32 ? INFINITY : (double)x; }
};
struct ConvF64Bits {
  __device__ double operator()(unsigned long long x) const {
    return __longlong_as_double((long long)x);
  }
};
struct ConvF64 {
  __device__ double operator()(double x) const { return x; }
};
struct ConvAlive {
  __device__ double operator()(uint8_t x) const { return x ? 1.0 : 0.0; }
};

// ===================================================================== host
// Ranks as host threads on one GPU: a thread that launches a kernel for the
// first time may make the driver load it (lazy loading), which waits for the
// whole device -- including a peer's barrier kernel that spins until this
// thread launches its own barrier.  So every host-launched barrier is preceded
// by a host rendezvous of the threads: a barrier kernel spins only after every
// rank has issued everything (and loaded every kernel) before it.
struct HostBarrier {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  bool failed = false;
  explicit HostBarrier(int w) : world(w) {}
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == world) {
      arrived = 0, ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || failed; });
    }
    if (failed) throw Error(SG_ECUDA, "a peer rank failed");
  }
  void fail() {
    std::lock_guard<std::mutex> lk(mu);
    failed = true;
    cv.notify_all();
  }
};

std::atomic<uint64_t> g_team_ids{0};
struct Team {
  uint64_t id = ++g_team_ids;
  int rank = 0, world = 1, device = 0;
  Layout lay;
  char *base = nullptr;
  char *peer[kMaxParts] = {};
  bool ipc[kMaxParts] = {};
  bool connected = false, poisoned = false;
  HostBarrier *host = nullptr;  // ranks as threads: rendezvous before device barriers
  TeamDev dev() const {
    TeamDev d{};
    for (int q = 0; q < world; ++q) d.base[q] = peer[q];
    d.rank = rank, d.world = world;
    return d;
  }
  ~Team() {
    cudaDeviceSynchronize();
    for (int q = 0; q < world; ++q)
      if (ipc[q] && peer[q]) cudaIpcCloseMemHandle(peer[q]);
    if (base) cudaFree(base);
  }
};

// mirror masks of one partition (cached on the partition graph)
struct MirrorInfo {
  uint64_t team_id = 0;
  DBuf<uint32_t> mask;    // [hi - lo]
  DBuf<uint32_t> any;     // [(hi - lo) / 32 + 1]
  int64_t lo = 0;
  Mirrors dev() const { return Mirrors{any.p, mask.p, lo}; }
  DBuf<uint32_t> mcount;  // [nv]: popc(mask) on owned rows, 0 elsewhere
};

const View &part_view(Graph &g) {
  switch (g.part.kind) {
    case 0: return g.csr;
    case 1: return g.csc();
    default: return g.sym();
  }
}
Cuts part_cuts(const Graph &g) {
  Cuts c{};
  c.D = g.part.world;
  for (int i = 0; i <= g.part.world; ++i) c.c[i] = g.part.cuts[(size_t)i];
  return c;
}

struct Stream {
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  Stream() {
    SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SG_CUDA(cudaEventCreate(&e0));
    SG_CUDA(cudaEventCreate(&e1));
  }
  ~Stream() {
    cudaStreamSynchronize(s);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
  }
};

void barrier(Team &T, cudaStream_t s) {
  if (T.host) T.host->wait();
  k_team_barrier<<<1, 32, 0, s>>>(T.dev(), nullptr);
  SG_CUDA(cudaGetLastError());
}

MirrorInfo &mirrors(Team &T, Graph &g, cudaStream_t s) {
  // cached on the partition graph, per team (the masks depend only on the cut)
  auto mi = std::static_pointer_cast<MirrorInfo>(g.part.mirrors);
  if (mi && mi->team_id == T.id) return *mi;
  mi = std::make_shared<MirrorInfo>();
  const View &v = part_view(g);
  const int64_t lo = g.part.lo, hi = g.part.hi;
  mi->team_id = T.id;
  mi->mask.alloc((size_t)std::max<int64_t>(hi - lo, 1));
  mi->any.alloc((size_t)((std::max<int64_t>(hi, lo + 1) - 1) / 32 - lo / 32 + 1));
  mi->lo = lo;
  SG_CUDA(cudaMemsetAsync(mi->any.p, 0, 4 * mi->any.n, s));
  mi->mcount.alloc((size_t)std::max<int64_t>(g.nv, 1));
  uint32_t *held = reinterpret_cast<uint32_t *>(T.base + T.lay.o_held);
  SG_CUDA(cudaMemsetAsync(held, 0, 4 * T.lay.nw, s));
  SG_CUDA(cudaMemsetAsync(mi->mcount.p, 0, 4 * mi->mcount.n, s));
  if (v.ne) k_px_held<<<grid_n(v.ne), 256, 0, s>>>(v.col.p, v.ne, lo, hi, held);
  SG_CUDA(cudaGetLastError());
  barrier(T, s);
  k_px_mask<<<grid_n(std::max<int64_t>(hi - lo, 1)), 256, 0, s>>>(T.dev(), T.lay, lo, hi,
                                                                    mi->mask.p, mi->any.p,
                                                                    mi->mcount.p);
  SG_CUDA(cudaGetLastError());
  barrier(T, s);
  SG_CUDA(cudaStreamSynchronize(s));
  g.part.mirrors = mi;
  return *mi;
}

// the run's loop as one WHILE node (body captured on s).  SG_PEER_EAGER=1
// (profiling only: ncu does not see kernels inside conditional nodes) runs
// the body from a host loop instead, one stream sync per round.
struct WhileGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  size_t nodes = 0;
  const bool eager = [] {
    const char *e = std::getenv("SG_PEER_EAGER");
    return e && std::atoi(e) != 0;
  }();
  const int uc = eager ? 0 : 1;  // Loop::use_cond of the body's kernels
  std::function<void(cudaGraphConditionalHandle)> body_;
  ~WhileGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
  template <class Body>
  void build(cudaStream_t s, Body &&body) {
    if (eager) {
      body_ = body;
      nodes = 0;
      return;
    }
    SG_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    SG_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    SG_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
    cudaGraph_t b = np.conditional.phGraph_out[0];
    SG_CUDA(cudaStreamBeginCaptureToGraph(s, b, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    try {
      body(cond);
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamEndCapture(s, &dummy);
      throw;
    }
    SG_CUDA(cudaStreamEndCapture(s, &b));
    SG_CUDA(cudaGraphGetNodes(b, nullptr, &nodes));
    SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  }
  void launch(cudaStream_t s, const Ctl *ctl) {
    if (!eager) {
      SG_CUDA(cudaGraphLaunch(exec, s));
      return;
    }
    for (;;) {
      body_(cudaGraphConditionalHandle{});
      int32_t done = 0;
      SG_CUDA(cudaMemcpyAsync(&done, &ctl->done, sizeof(done), cudaMemcpyDeviceToHost, s));
      SG_CUDA(cudaStreamSynchronize(s));
      if (done) break;
    }
  }
};

struct Out {
  double *labels_out;
  sg_round *rounds_out;
  int64_t cap;
  int64_t *nrounds;
  double *ms_out;
};

void finish_run(Team &T, Stream &S, RunBufs &rb, double *labels_d, int64_t nv, const Out &o,
                int64_t max_rounds, size_t body_nodes) {
  SG_CUDA(cudaEventSynchronize(S.e1));
  float ms = 0;
  SG_CUDA(cudaEventElapsedTime(&ms, S.e0, S.e1));
  if (o.ms_out) *o.ms_out = ms;
  Ctl h;
  SG_CUDA(cudaMemcpy(&h, rb.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
  Hdr hh;
  SG_CUDA(cudaMemcpy(&hh, T.base, sizeof(Hdr), cudaMemcpyDeviceToHost));
  if (hh.err || h.error == SG_ECUDA) {
    T.poisoned = true;
    throw Error(SG_ECUDA, std::string("peer barrier timed out: a rank did not arrive within 60 s "
                          "(the team is unusable; create a new one)") +
                          (T.host ? "; ranks as threads share one GPU's hardware queues: set "
                                    "CUDA_DEVICE_MAX_CONNECTIONS >= world + 2 before CUDA starts"
                                  : ""));
  }
  const int64_t rounds = h.round;
  g_launches.fetch_add((int64_t)body_nodes * rounds, std::memory_order_relaxed);
  std::vector<RoundStat> st((size_t)std::min<int64_t>(rounds, rb.stats_cap));
  if (!st.empty())
    SG_CUDA(cudaMemcpy(st.data(), rb.stats.p, sizeof(RoundStat) * st.size(),
                       cudaMemcpyDeviceToHost));
  if (o.rounds_out && !st.empty())
    std::memcpy(o.rounds_out, st.data(),
                sizeof(RoundStat) * (size_t)std::min<int64_t>(o.cap, (int64_t)st.size()));
  *o.nrounds = rounds;
  if (o.labels_out)
    SG_CUDA(cudaMemcpy(o.labels_out, labels_d, sizeof(double) * nv, cudaMemcpyDeviceToHost));
  if (h.error == SG_ECONVERGE)
    throw Error(SG_ECONVERGE, "did not converge within " + std::to_string(max_rounds) + " rounds");
  if (h.error) throw Error(h.error, "round log capacity exhausted");
}

// --------------------------------------------------------- push driver --
template <int KIND>
void run_peer_push(Team &T, Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds,
                   const Out &o) {
  using Op = BmMin<KIND>;
  using L = typename Op::L;
  const bool cc = p.app == SG_APP_CC;
  const bool classic = (p.flags & SG_FLAG_TWC_CLASSIC) != 0;
  const View &v = part_view(g);
  const int64_t nv = v.nv;
  const Cuts cuts = part_cuts(g);
  const uint32_t *inv = g.part.relabeled ? g.part.inv.p : nullptr;
  const int R = T.rank;
  const uint32_t lo = (uint32_t)cuts.c[R], hi = (uint32_t)cuts.c[R + 1];
  // edgeless tail of the block (relabeled push / symmetrized partitions)
  const uint32_t zlo = g.part.zlo >= (int64_t)lo && g.part.zlo <= (int64_t)hi ? (uint32_t)g.part.zlo : hi;
  Stream S;
  cudaStream_t s = S.s;
  MirrorInfo &mi = mirrors(T, g, s);
  RunBufs rb;
  rb.alloc_common(nv, stats_cap(max_rounds));
  PushArgs a = rb.push_args(v, thr);
  a.q[1] = a.q[0];  // the frontier is rebuilt by k_px_compact after the round's relaxations
  a.dense_lo = lo, a.dense_n = hi - lo;
  a.sched = p.sched == SG_SCHED_LB ? 1 : p.sched == SG_SCHED_VERTEX ? 2 : p.sched == SG_SCHED_EDGE ? 3 : 0;
  const TeamDev td = T.dev();
  L *lab = reinterpret_cast<L *>(T.base + T.lay.o_d[0]);
  uint32_t *nb = reinterpret_cast<uint32_t *>(T.base + T.lay.o_nb);
  DBuf<L> snap(std::max<int64_t>(hi - lo, 1));
  DBuf<long long> acc(kSlot), tsum((nv + kFT - 1) / kFT + 1);
  DBuf<uint32_t> tick(2);  // last-block tickets of reduce / compact
  DBuf<double> out(std::max<int64_t>(nv, 1));
  const bool weighted = p.app == SG_APP_SSSP && g.weighted;
  const Op op{lab, KIND == 2 ? g.w32.p : nullptr, KIND == 3 && weighted ? g.w64.p : nullptr,
              snap.p, nb};
  int64_t src = p.source;  // in the partition's numbering
  if (!cc && inv) {
    uint32_t x = 0;
    SG_CUDA(cudaMemcpy(&x, inv + p.source, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    src = x;
  }
  const bool owns_src = !cc && src >= lo && src < hi;
  const L inf = sizeof(L) == 4 ? (L)kInf32 : (L)0x7ff0000000000000ull;
  Ctl *ctl = rb.ctl.p;
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  Launcher Lc;
  WhileGraph W;
  W.build(s, [&](cudaGraphConditionalHandle cond) {
    const Loop lp{limit, max_rounds, cond, W.uc};
    RoundCtx c{Lc, s, cond, W.uc};
    bm_round(c, a, op, p.blocked != 0, classic, tsum.p, /*compact=*/false);
    // reduce (+ barrier in its last block), compact (+ publish, barrier, advance)
    Lc.go("peer_reduce", k_px_reduce<L>, ticket_grid((int64_t)T.lay.nw, 4), 256, s, td, T.lay, cuts,
          ctl, acc.p, tick.p);
    Lc.go("peer_compact", k_px_compact<L>, ticket_grid(std::max<int64_t>(hi - lo, 1), 8), 256, s, td,
          T.lay, cuts, a, mi.dev(), rb.q0.p, snap.p, acc.p, tick.p + 1, lp, zlo);
  });
  SG_CUDA(cudaEventRecord(S.e0, s));
  Lc.go("init", k_ctl_init, 1, 1, s, ctl, (int32_t)cc, cc ? hi - lo : (owns_src ? 1u : 0u));
  fill<uint32_t>(Lc, nb, (int64_t)T.lay.nw, 0u, s);
  fill<long long>(Lc, acc.p, kSlot, 0ll, s);
  fill<uint32_t>(Lc, tick.p, 2, 0u, s);
  if (cc && inv) {  // relabeled: a vertex's label is its original id (perm)
    Lc.go("init", k_copy_as<L>, grid_n(nv), 256, s, (const uint32_t *)g.part.perm.p, nv, lab);
    Lc.go("init", k_copy_as<L>, grid_n(hi - lo), 256, s, (const uint32_t *)g.part.perm.p + lo,
          (int64_t)(hi - lo), snap.p);
  } else if (cc) {  // cc: label = id; round 0 is every owned row (dense), snapshot = id
    Lc.go("init", k_iota_from<L>, grid_n(nv), 256, s, lab, nv, (int64_t)0);
    Lc.go("init", k_iota_from<L>, grid_n(hi - lo), 256, s, snap.p, (int64_t)(hi - lo), (int64_t)lo);
  } else {
    fill<L>(Lc, lab, nv, inf, s);
    Lc.go("init", k_set1<L>, 1, 1, s, lab, src, (L)0);
    if (owns_src) {
      Lc.go("init", k_set1<uint32_t>, 1, 1, s, rb.q0.p, (int64_t)0, (uint32_t)src);
      Lc.go("init", k_set1<L>, 1, 1, s, snap.p, (int64_t)0, (L)0);
    }
  }
  barrier(T, s);  // every region initialised before any peer writes into it
  W.launch(s, ctl);
  barrier(T, s);
  if (sizeof(L) == 4)
    k_px_gather<uint32_t><<<grid_n(nv), 256, 0, s>>>(td, T.lay.o_d[0], cuts, nv, inv, out.p,
                                                     ConvU32{});
  else
    k_px_gather<unsigned long long><<<grid_n(nv), 256, 0, s>>>(td, T.lay.o_d[0], cuts, nv, inv,
                                                              out.p, ConvF64Bits{});
  SG_CUDA(cudaGetLastError());
  barrier(T, s);  // nobody re-initialises its region while a peer still gathers from it
  SG_CUDA(cudaEventRecord(S.e1, s));
  finish_run(T, S, rb, out.p, nv, o, max_rounds, W.nodes);
}

// ---------------------------------------------------------- bfs driver --
void run_peer_bfs(Team &T, Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds,
                  const Out &o) {
  const bool classic = (p.flags & SG_FLAG_TWC_CLASSIC) != 0;
  const View &v = part_view(g);
  const int64_t nv = v.nv;
  const Cuts cuts = part_cuts(g);
  const uint32_t *inv = g.part.relabeled ? g.part.inv.p : nullptr;
  const int R = T.rank;
  const uint32_t lo = (uint32_t)cuts.c[R], hi = (uint32_t)cuts.c[R + 1];
  // edgeless tail of the block (relabeled push / symmetrized partitions)
  const uint32_t zlo = g.part.zlo >= (int64_t)lo && g.part.zlo <= (int64_t)hi ? (uint32_t)g.part.zlo : hi;
  Stream S;
  cudaStream_t s = S.s;
  MirrorInfo &mi = mirrors(T, g, s);
  RunBufs rb;
  rb.alloc_common(nv, stats_cap(max_rounds));
  PushArgs a = rb.push_args(v, thr);
  a.q[1] = a.q[0];  // the frontier is rebuilt by k_px_bfs_compact after the relaxations
  a.sched = p.sched == SG_SCHED_LB ? 1 : p.sched == SG_SCHED_VERTEX ? 2 : p.sched == SG_SCHED_EDGE ? 3 : 0;
  const TeamDev td = T.dev();
  uint32_t *lab = reinterpret_cast<uint32_t *>(T.base + T.lay.o_d[0]);
  uint32_t *vis = reinterpret_cast<uint32_t *>(T.base + T.lay.o_nb);
  uint32_t *prev = reinterpret_cast<uint32_t *>(T.base + T.lay.o_prev);
  DBuf<long long> acc(kSlot), tsum((nv + kFT - 1) / kFT + 1);
  DBuf<uint32_t> tick(2);  // last-block tickets of reduce / compact
  DBuf<double> out(std::max<int64_t>(nv, 1));
  int64_t src = p.source;
  if (inv) {
    uint32_t x = 0;
    SG_CUDA(cudaMemcpy(&x, inv + p.source, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    src = x;
  }
  const bool owns_src = src >= lo && src < hi;
  // prev is the round-start copy the operator's compaction would advance; the
  // peer compaction advances it instead (BmBfs::take is not used)
  const BmBfs op{lab, vis, prev};
  Ctl *ctl = rb.ctl.p;
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  Launcher Lc;
  WhileGraph W;
  W.build(s, [&](cudaGraphConditionalHandle cond) {
    const Loop lp{limit, max_rounds, cond, W.uc};
    RoundCtx c{Lc, s, cond, W.uc};
    bm_round(c, a, op, p.blocked != 0, classic, tsum.p, /*compact=*/false);
    // reduce (+ barrier in its last block), compact (+ publish, barrier, advance)
    Lc.go("peer_reduce", k_px_bfs_reduce, ticket_grid((int64_t)T.lay.nw, 4), 256, s, td, T.lay, cuts,
          ctl, acc.p, tick.p);
    Lc.go("peer_compact", k_px_bfs_compact, ticket_grid(std::max<int64_t>(hi - lo, 1), 8), 256, s, td,
          T.lay, cuts, a, mi.dev(), rb.q0.p, acc.p, tick.p + 1, lp, zlo);
  });
  SG_CUDA(cudaEventRecord(S.e0, s));
  Lc.go("init", k_ctl_init, 1, 1, s, ctl, 0, owns_src ? 1u : 0u);
  fill<uint32_t>(Lc, vis, (int64_t)T.lay.nw, 0u, s);
  fill<uint32_t>(Lc, prev, (int64_t)T.lay.nw, 0u, s);
  fill<long long>(Lc, acc.p, kSlot, 0ll, s);
  fill<uint32_t>(Lc, tick.p, 2, 0u, s);
  fill<uint32_t>(Lc, lab, nv, kInf32, s);
  // every rank knows the source is visited (its label 0 is final)
  Lc.go("init", k_set1<uint32_t>, 1, 1, s, lab, src, 0u);
  Lc.go("init", k_set1<uint32_t>, 1, 1, s, vis, src >> 5, 1u << (src & 31));
  Lc.go("init", k_set1<uint32_t>, 1, 1, s, prev, src >> 5, 1u << (src & 31));
  if (owns_src) Lc.go("init", k_set1<uint32_t>, 1, 1, s, rb.q0.p, (int64_t)0, (uint32_t)src);
  barrier(T, s);
  W.launch(s, ctl);
  barrier(T, s);
  k_px_gather<uint32_t><<<grid_n(nv), 256, 0, s>>>(td, T.lay.o_d[0], cuts, nv, inv, out.p,
                                                   ConvU32{});
  SG_CUDA(cudaGetLastError());
  barrier(T, s);
  SG_CUDA(cudaEventRecord(S.e1, s));
  finish_run(T, S, rb, out.p, nv, o, max_rounds, W.nodes);
}

// ----------------------------------------------------------- pr driver --
void run_peer_pr(Team &T, Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds,
                 const Out &o) {
  const View &v = part_view(g);  // this rank's CSC rows
  const int64_t nv = v.nv;
  const Cuts cuts = part_cuts(g);
  const uint32_t *pinv = g.part.relabeled ? g.part.inv.p : nullptr;  // old -> new id
  const int R = T.rank;
  const uint32_t lo = (uint32_t)cuts.c[R], hi = (uint32_t)cuts.c[R + 1];
  // everything that may synchronise the device (layout builds) comes before
  // the first barrier: with ranks as threads a device-wide sync would wait on
  // a peer's spinning barrier kernel
  const int64_t hs = exact_hs();
  const ExactLayout &XL = g.exact(hs, lo, hi);
  Stream S;
  cudaStream_t s = S.s;
  MirrorInfo &mi = mirrors(T, g, s);
  RunBufs rb;
  rb.alloc_common(nv, stats_cap(max_rounds));
  PullArgs a = rb.pull_args(v, thr, 0);
  a.row_lo = lo, a.row_n = hi - lo;
  a.mcount = mi.mcount.p;
  const TeamDev td = T.dev();
  double *aux0 = reinterpret_cast<double *>(T.base + T.lay.o_d[0]);
  double *aux1 = reinterpret_cast<double *>(T.base + T.lay.o_d[1]);
  double *rank = reinterpret_cast<double *>(T.base + T.lay.o_d[2]);
  DBuf<double> inv(std::max<int64_t>(nv, 1)), hacc(1), out(std::max<int64_t>(nv, 1));
  DBuf<unsigned long long> gmax(1);
  DBuf<long long> acc(kSlot);
  DBuf<uint32_t> head(1);
  const double d = p.damping, omd = 1.0 - p.damping;
  PrOp op{aux0, aux1, aux1, aux0, rank, inv.p, d, omd};
  op.mcount = a.mcount;
  PrFold fold{aux0, aux1, aux1, aux0, rank, inv.p, d, omd, a.mcount};
  Cuts one{};
  one.D = 1, one.c[0] = 0, one.c[1] = nv;
  Ctl *ctl = rb.ctl.p;
  std::vector<std::unique_ptr<DBuf<char>>> keep;
  PrxArgs xa = prx_args(v, XL, std::max<int64_t>(thr, hs), thr != kNoHuge, ctl, nullptr, gmax.p,
                        head.p, [&](size_t bytes) {
                          keep.emplace_back(new DBuf<char>(bytes));
                          return (void *)keep.back()->p;
                        });
  const int gx = occupancy_grid(k_prx<0>, kTB);
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  Launcher L;
  WhileGraph W;
  W.build(s, [&](cudaGraphConditionalHandle cond) {
    const Loop lp{limit, max_rounds, cond, W.uc};
    // acc = {twc launches, lb launches, nhuge, huge_edges, nlarge, large_edges}, then
    // acc[6] = max |delta| bits, acc[7] = comm_broadcast -- summed / maxed over ranks
    PrStop st2{gmax.p, d, p.tol, g.part.full_ne, limit, max_rounds, cond, W.uc, 1, 2, acc.p};
    L.go("pr_pull", k_prx<0>, gx, kTB, s, xa, fold);
    // round r writes aux1 when r is even, aux0 when odd (PrFold)
    L.go("peer_rows", k_px_rows<double>, grid_n(std::max<int64_t>(hi - lo, 1) / 32 + 1), 256, s, td,
         T.lay.o_d[1], T.lay.o_d[0], 0, (const Ctl *)ctl, (int64_t)lo, (int64_t)hi, mi.dev());
    L.go("peer_sync", k_px_pr_sync, 1, 32, s, td, ctl, (int)(hi > lo), acc.p);
    L.go("pr_finish", k_pull_finish<PrOp, true>, 1, 1024, s, a, op, hacc.p, st2);
    fill<uint32_t>(L, head.p, 1, 0u, s);
    L.go("guard", k_loop_guard, 1, 32, s, (const Ctl *)ctl, lp);
  });
  SG_CUDA(cudaEventRecord(S.e0, s));
  L.go("init", k_ctl_init, 1, 1, s, ctl, 1, (uint32_t)nv);
  L.go("init", k_pr_init, grid_n(nv), 256, s, (const int64_t *)g.csr.off.p, nv, omd, inv.p, rank,
       aux0);
  L.go("init", k_copy_f64, grid_n(nv), 256, s, (const double *)aux0, nv, aux1);
  fill<unsigned long long>(L, gmax.p, 1, 0ull, s);
  fill<long long>(L, acc.p, kSlot, 0ll, s);
  fill<uint32_t>(L, head.p, 1, 0u, s);
  fill<uint32_t>(L, xa.ck_meta, xa.nchunks, 0u, s);
  if (xa.nsplit) {
    L.go("init", k_prx_chunks, 1, 1024, s, xa.off, xa.big, xa.nsplit, (uint32_t *)xa.ck_first,
         (uint32_t *)xa.ck_row);
    L.go("pr_guess", k_prx_guess_sums, grid_n((int64_t)xa.nchunks * 32, kTB), kTB, s, xa,
         (const double *)inv.p);
    L.go("pr_guess", k_prx_guess_scan, grid_n((int64_t)xa.nsplit * 32, kTB), kTB, s, xa);
  }
  if (v.ne) {  // gain: exact sums of this rank's rows
    PrxArgs xg = xa;
    xg.gain = 1;
    L.go("pr_gain", k_prx<0>, gx, kTB, s, xg, fold);
  }
  // ... then the maximum over ranks (eps_stop, apps.py:164-171)
  L.go("peer_publish", k_px_publish, 1, 256, s, td, (const Ctl *)nullptr,
       (const long long *)gmax.p, 1);
  barrier(T, s);
  L.go("peer_sum", k_px_reduce_slots, 1, 32, s, td, (const Ctl *)nullptr,
       (long long *)gmax.p, 1, 1u);
  fill<uint32_t>(L, head.p, 1, 0u, s);
  if (xa.nsplit) {
    L.go("pr_guess", k_prx_guess_sums, grid_n((int64_t)xa.nchunks * 32, kTB), kTB, s, xa,
         (const double *)aux0);
    L.go("pr_guess", k_prx_guess_scan, grid_n((int64_t)xa.nsplit * 32, kTB), kTB, s, xa);
  }
  L.go("init", k_static_bins, grid_n(hi - lo), 256, s, v.off.p, lo, hi - lo, thr, rb.largeq.p,
       rb.hugeq.p, ctl, one);
  barrier(T, s);  // gain slots read everywhere, every region initialised
  W.launch(s, ctl);
  barrier(T, s);
  k_px_gather<double><<<grid_n(nv), 256, 0, s>>>(td, T.lay.o_d[2], cuts, nv, pinv, out.p,
                                                  ConvF64{});
  SG_CUDA(cudaGetLastError());
  barrier(T, s);
  SG_CUDA(cudaEventRecord(S.e1, s));
  finish_run(T, S, rb, out.p, nv, o, max_rounds, W.nodes);
}

// -------------------------------------------------------- kcore driver --
void run_peer_kcore(Team &T, Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds,
                    const Out &o) {
  const bool classic = (p.flags & SG_FLAG_TWC_CLASSIC) != 0;
  const View &v = part_view(g);  // this rank's symmetrized rows
  const int64_t nv = v.nv;
  const Cuts cuts = part_cuts(g);
  const uint32_t *inv = g.part.relabeled ? g.part.inv.p : nullptr;
  const int R = T.rank;
  const uint32_t lo = (uint32_t)cuts.c[R], hi = (uint32_t)cuts.c[R + 1];
  Stream S;
  cudaStream_t s = S.s;
  MirrorInfo &mi = mirrors(T, g, s);
  RunBufs rb;
  rb.alloc_common(nv, stats_cap(max_rounds));
  rb.dying.alloc(std::max<int64_t>(nv, 1));
  PullArgs a = rb.pull_args(v, thr, 1);
  // relabeled: [zlo, hi) are the block's isolated vertices -- they die in
  // round 0 with no neighbour to tell, so they are killed at init and only
  // counted in round 0's log (Ctl::fzero), as on one GPU; the dense pass
  // stops at zlo
  const uint32_t zlo = g.part.zlo >= (int64_t)lo && g.part.zlo <= (int64_t)hi ? (uint32_t)g.part.zlo : hi;
  a.row_lo = lo, a.row_n = zlo - lo;
  a.mcount = mi.mcount.p;
  PushArgs w = rb.push_args(v, kNoHuge);
  w.src_mode = 1;
  w.no_enqueue = 1;  // marks only; owners collect them after the barrier
  const TeamDev td = T.dev();
  uint8_t *alive = reinterpret_cast<uint8_t *>(T.base + T.lay.o_d[0]);
  uint32_t *mark = reinterpret_cast<uint32_t *>(T.base + T.lay.o_d[1]);
  DBuf<uint32_t> hcnt(std::max<int64_t>(nv, 1));
  DBuf<double> out(std::max<int64_t>(nv, 1));
  DBuf<long long> acc(kSlot);
  const KcOp op{alive, (uint32_t)std::min<int64_t>(p.k, 0xffffffffLL)};
  OpMarkPeer mop{alive, mark, td, T.lay.o_d[1], cuts};
  Ctl *ctl = rb.ctl.p;
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  Launcher L;
  WhileGraph W;
  W.build(s, [&](cudaGraphConditionalHandle cond) {
    const Loop lp{limit, max_rounds, cond, W.uc};
    RoundCtx c{L, s, cond, W.uc};
    pull_round(c, a, op, p.blocked != 0, hcnt.p, classic);
    if (thr != kNoHuge)
      L.go("kcore_huge", k_pull_finish<KcOp, false>, 1, 1024, s, a, op, hcnt.p, PrStop{});
    L.go("kcore_kill", k_kcore_kill, grid_n(nv), 256, s, a, alive);
    L.go("dist", k_dist_kc_collect, 1, 32, s, a, acc.p);
    L.go("kcore_stats", k_kcore_reset, 1, 1, s, a);
    L.go("mark_twc", k_push_twc<OpMarkPeer>, occupancy_grid(k_push_twc<OpMarkPeer>, kTB), kTB, s,
         w, mop);
    L.go("mark_large", k_push_large<OpMarkPeer>, occupancy_grid(k_push_large<OpMarkPeer>, kTB),
         kTB, s, w, mop);
    // every rank has counted (reads of mirrors' alive flags) and marked
    L.go("peer_barrier", k_team_barrier, 1, 32, s, td, ctl);
    // the round's deaths -> the mirror holders (read by the next round's count)
    L.go("peer_kill", k_px_kill, grid_n(hi - lo), 256, s, td, T.lay, (const Ctl *)ctl,
         (const uint32_t *)rb.dying.p, mi.dev());
    L.go("dist", k_px_kc_compact, grid_n(((int64_t)hi - lo) / 4 + 1), 256, s, (const Ctl *)ctl,
         (const uint32_t *)mark, (const uint8_t *)alive, lo, hi, rb.q0.p, rb.q1.p, &ctl->nsize);
    L.go("dist", k_dist_kc_next, 1, 32, s, (const Ctl *)ctl, acc.p);
    L.go("peer_publish", k_px_publish, 1, 256, s, td, (const Ctl *)ctl, (const long long *)acc.p,
         kDistN);
    L.go("peer_barrier", k_team_barrier, 1, 32, s, td, ctl);
    L.go("peer_sum", k_px_reduce_slots, 1, 32, s, td, (const Ctl *)ctl, acc.p, kDistN, 0u);
    L.go("advance", k_dist_kc_advance, 1, 32, s, a, acc.p, lp);
    L.go("guard", k_loop_guard, 1, 32, s, (const Ctl *)ctl, lp);
  });
  SG_CUDA(cudaEventRecord(S.e0, s));
  L.go("init", k_ctl_init, 1, 1, s, ctl, 1, hi - lo);
  fill<uint8_t>(L, alive, nv, (uint8_t)1, s);
  if (zlo < hi) {
    fill<uint8_t>(L, alive + zlo, (int64_t)(hi - zlo), (uint8_t)0, s);
    L.go("init", k_set1<uint32_t>, 1, 1, s, &ctl->fzero, (int64_t)0, hi - zlo);
  }
  fill<uint32_t>(L, mark, nv, 0u, s);
  fill<uint32_t>(L, hcnt.p, nv, 0u, s);
  fill<long long>(L, acc.p, kSlot, 0ll, s);
  barrier(T, s);
  W.launch(s, ctl);
  barrier(T, s);
  k_px_gather<uint8_t><<<grid_n(nv), 256, 0, s>>>(td, T.lay.o_d[0], cuts, nv, inv, out.p,
                                                   ConvAlive{});
  SG_CUDA(cudaGetLastError());
  barrier(T, s);
  SG_CUDA(cudaEventRecord(S.e1, s));
  finish_run(T, S, rb, out.p, nv, o, max_rounds, W.nodes);
}

int part_kind_of(int app) {
  return app == SG_APP_PR ? 1 : (app == SG_APP_CC || app == SG_APP_KCORE) ? 2 : 0;
}

// Load the kernels a rank launches right after passing a barrier before any
// team runs: under lazy module loading a first launch may wait on the device,
// where a peer's barrier kernel spins until this rank arrives (seen as a
// cold-process barrier timeout with ranks as threads on one GPU).  The
// round kernels are loaded when the run's graph is instantiated.
void preload_peer_kernels() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncAttributes fa;
    const void *ks[] = {
        (const void *)k_team_barrier,
        (const void *)k_px_held,
        (const void *)k_px_mask,
        (const void *)k_px_gather<uint32_t, ConvU32>,
        (const void *)k_px_gather<unsigned long long, ConvF64Bits>,
        (const void *)k_px_gather<double, ConvF64>,
        (const void *)k_px_gather<uint8_t, ConvAlive>,
    };
    for (const void *k : ks) SG_CUDA(cudaFuncGetAttributes(&fa, k));
  });
}

void team_run(Team &T, Graph &g, const sg_params &p, const Out &o) {
  preload_peer_kernels();
  if (!T.connected) throw Error(SG_ECONFIG, "team not connected (sg_team_connect)");
  if (T.poisoned) throw Error(SG_ECUDA, "team unusable after a barrier timeout");
  if (!g.is_part()) throw Error(SG_ECONFIG, "sg_team_run needs an edge-cut partition (sg_graph_partition)");
  if (p.app < SG_APP_BFS || p.app > SG_APP_KCORE) throw Error(SG_ECONFIG, "unknown app");
  if (g.part.world != T.world || g.part.rank != T.rank)
    throw Error(SG_ECONFIG, "partition " + std::to_string(g.part.rank) + "/" +
                                std::to_string(g.part.world) + " run by team rank " +
                                std::to_string(T.rank) + "/" + std::to_string(T.world));
  if (g.nv != T.lay.nv) throw Error(SG_ECONFIG, "team region sized for another vertex count");
  if (g.part.kind != part_kind_of(p.app))
    throw Error(SG_ECONFIG, std::string("app needs the ") +
                                (part_kind_of(p.app) == 0 ? "CSR" : part_kind_of(p.app) == 1 ? "CSC" : "symmetrized") +
                                " partition (sg_graph_partition kind " +
                                std::to_string(part_kind_of(p.app)) + ")");
  if ((p.app == SG_APP_BFS || p.app == SG_APP_SSSP) && (p.source < 0 || p.source >= g.nv))
    throw Error(SG_ECONFIG, "source " + std::to_string(p.source) + " outside graph");
  if (p.app == SG_APP_SSSP && g.weighted && g.wmin < 0)
    throw Error(SG_ECONFIG, "sssp requires non-negative weights");
  if (p.app == SG_APP_PR && !(p.damping > 0.0 && p.damping < 1.0))
    throw Error(SG_ECONFIG, "damping must be in (0, 1)");
  if (p.app == SG_APP_PR && !(p.tol > 0.0)) throw Error(SG_ECONFIG, "tolerance must be positive");
  if (p.app == SG_APP_KCORE && p.k < 1) throw Error(SG_ECONFIG, "k must be >= 1");
  if (p.sched < SG_SCHED_ALB || p.sched > SG_SCHED_EDGE) throw Error(SG_ECONFIG, "unknown scheduler");
  if (p.devices != T.world) throw Error(SG_ECONFIG, "params.devices must equal the team size");
  const int64_t max_rounds =
      p.max_rounds > 0 ? p.max_rounds : 10 * std::max<int64_t>(g.nv, 1) + 256;
  const int64_t thr = p.sched == SG_SCHED_TWC ? kNoHuge
                      : p.sched == SG_SCHED_ALB ? std::max<int64_t>(1, p.threshold)
                                                : 1;  // lb / vertex / edge: the LB path
  *o.nrounds = 0;
  if (o.ms_out) *o.ms_out = 0.0;
  if (g.nv == 0) return;
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev));
  if (dev != T.device) throw Error(SG_ECONFIG, "team created on another device");
  if (p.app == SG_APP_PR) return run_peer_pr(T, g, p, thr, max_rounds, o);
  if (p.app == SG_APP_KCORE) return run_peer_kcore(T, g, p, thr, max_rounds, o);
  if (p.app == SG_APP_CC) return run_peer_push<0>(T, g, p, thr, max_rounds, o);
  const bool weighted = p.app == SG_APP_SSSP && g.weighted;
  if (p.app == SG_APP_BFS) return run_peer_bfs(T, g, p, thr, max_rounds, o);
  if (!weighted) return run_peer_push<1>(T, g, p, thr, max_rounds, o);  // unit-weight sssp
  const double bound = (double)g.wmax * (double)std::max<int64_t>(g.nv - 1, 1);
  if (g.w32.p && bound < 4294967295.0) return run_peer_push<2>(T, g, p, thr, max_rounds, o);
  return run_peer_push<3>(T, g, p, thr, max_rounds, o);
}

// ------------------------------------------ block-local relabel (partition) --
__global__ void k_px_indeg(const uint32_t *col, int64_t ne, uint32_t *cnt) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += st)
    atomicAdd(cnt + col[e], 1u);
}
// key = block << 32 | ~total degree: an ascending stable sort puts every block
// onto itself, highest degree first, ties by id
__global__ void k_px_key(const int64_t *off, const uint32_t *indeg, int64_t nv, Cuts cuts,
                         unsigned long long *key, uint32_t *ids) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st) {
    const unsigned long long d = (unsigned long long)(off[v + 1] - off[v]) + indeg[v];
    const unsigned long long dd = d > 0xffffffffull ? 0xffffffffull : d;
    key[v] = ((unsigned long long)owner_of(cuts, (uint32_t)v) << 32) | (0xffffffffull - dd);
    ids[v] = (uint32_t)v;
  }
}
// second pass: the first kb vertices of each block (by degree) keep their
// degree order, the rest follow in id order (a full degree order also
// reorders the frontier and loses ~10 % on rmat24: profiles/r2x_hotk_sweep),
// and with `off` (push / symmetrized views) the rest without rows go last;
// nz counts those of block `rank`
__global__ void k_px_key2(const uint32_t *perm0, int64_t nv, Cuts cuts, int64_t kb,
                          const int64_t *off, int rank, unsigned long long *key, uint32_t *ids,
                          unsigned long long *nz) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += st) {
    const uint32_t v = perm0[i];
    const int b = owner_of(cuts, v);
    const long long pos = i - cuts.c[b];
    unsigned long long cls = 0, low = (unsigned long long)pos;
    if (pos >= kb) {
      cls = off && off[v + 1] == off[v] ? 2 : 1;
      low = v;
      if (cls == 2 && b == rank) atomicAdd(nz, 1ull);
    }
    key[i] = ((unsigned long long)b << 34) | (cls << 32) | low;
    ids[i] = v;
  }
}
__global__ void k_px_invert(const uint32_t *perm, int64_t nv, uint32_t *inv) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += st)
    inv[perm[i]] = (uint32_t)i;
}
// len[i] = degree of old row perm[i] for new rows i in [lo, hi), 0 elsewhere
__global__ void k_px_len(const int64_t *off, const uint32_t *perm, int64_t nv, int64_t lo,
                         int64_t hi, int64_t *len) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nv; i += st) {
    int64_t d = 0;
    if (i >= lo && i < hi) {
      const uint32_t o = perm[i];
      d = off[o + 1] - off[o];
    }
    len[i] = d;
  }
}
// new row i = old row perm[i], ids renamed, in-row order kept (pr sums in it);
// one warp per row
__global__ void k_px_copy_rows(const int64_t *off, const uint32_t *col, const int64_t *w64,
                               const uint32_t *perm, const uint32_t *inv, int64_t lo, int64_t hi,
                               const int64_t *noff, uint32_t *ncol, int64_t *nw64) {
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < hi;
       i += warps) {
    const uint32_t o = perm[i];
    const int64_t s = off[o], d = off[o + 1] - s, t = noff[i];
    for (int64_t j = lane_id(); j < d; j += 32) {
      ncol[t + j] = inv[col[s + j]];
      if (nw64) nw64[t + j] = w64[s + j];
    }
  }
}

// ------------------------------------------------------------ partition --
__global__ void k_part_off(const int64_t *off, int64_t nv, int64_t lo, int64_t hi, int64_t *out) {
  const int64_t base = off[lo], top = off[hi];
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= nv; v += st) {
    const int64_t x = off[v];
    out[v] = (x < base ? base : x > top ? top : x) - base;
  }
}

void slice_view(View &out, const View &in, int64_t lo, int64_t hi, int64_t *e0, int64_t *e1) {
  out.nv = in.nv;
  out.off.alloc((size_t)in.nv + 1);
  k_part_off<<<grid_n(in.nv + 1), 256>>>(in.off.p, in.nv, lo, hi, out.off.p);
  SG_CUDA(cudaGetLastError());
  SG_CUDA(cudaMemcpy(e0, in.off.p + lo, sizeof(int64_t), cudaMemcpyDeviceToHost));
  SG_CUDA(cudaMemcpy(e1, in.off.p + hi, sizeof(int64_t), cudaMemcpyDeviceToHost));
  out.ne = *e1 - *e0;
  out.col.alloc((size_t)std::max<int64_t>(out.ne, 1));
  if (out.ne)
    SG_CUDA(cudaMemcpy(out.col.p, in.col.p + *e0, sizeof(uint32_t) * out.ne,
                       cudaMemcpyDeviceToDevice));
}

// default: relabel skewed graphs of >= 2^20 vertices (as the single-device store)
bool want_part_relabel(Graph &g, int mode) {
  if (mode > 0) return true;
  if (mode < 0) return false;
  return g.nv >= ((int64_t)1 << 20) && g.top1_share() >= 0.10;
}

// the block-local relabeled rows [lo, hi) of view v (+ weights for kind 0)
void relabeled_slice(Graph &g, const View &v, int kind, const Cuts &c, Graph &P) {
  const int64_t nv = g.nv, lo = P.part.lo, hi = P.part.hi;
  P.part.relabeled = true;
  P.part.perm.alloc((size_t)std::max<int64_t>(nv, 1));
  P.part.inv.alloc((size_t)std::max<int64_t>(nv, 1));
  {
    DBuf<uint32_t> indeg(nv), ids(nv);
    DBuf<unsigned long long> key(nv), key2(nv);
    SG_CUDA(cudaMemset(indeg.p, 0, sizeof(uint32_t) * nv));
    if (v.ne) k_px_indeg<<<grid_n(v.ne), 256>>>(v.col.p, v.ne, indeg.p);
    k_px_key<<<grid_n(nv), 256>>>(v.off.p, indeg.p, nv, c, key.p, ids.p);
    SG_CUDA(cudaGetLastError());
    int bbits = 0;
    while ((1ll << bbits) < c.D) ++bbits;
    size_t tb = 0, tb2 = 0;
    DBuf<uint32_t> perm0(nv);
    SG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, ids.p, perm0.p, (int)nv,
                                            0, 32 + bbits));
    SG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, key.p, key2.p, ids.p, P.part.perm.p,
                                            (int)nv, 0, 34 + bbits));
    DBuf<char> t(std::max<size_t>(std::max(tb, tb2), 1));
    SG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, key.p, key2.p, ids.p, perm0.p, (int)nv, 0,
                                            32 + bbits));
    // hot set per block: the single-device store's 2^16 spread over the ranks
    const int64_t kb = std::max<int64_t>(1024, ((int64_t)1 << 16) / c.D);
    DBuf<unsigned long long> nz(1);
    SG_CUDA(cudaMemset(nz.p, 0, sizeof(unsigned long long)));
    k_px_key2<<<grid_n(nv), 256>>>(perm0.p, nv, c, kb, kind == 1 ? nullptr : v.off.p,
                                   P.part.rank, key.p, ids.p, nz.p);
    SG_CUDA(cudaGetLastError());
    SG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb2, key.p, key2.p, ids.p, P.part.perm.p,
                                            (int)nv, 0, 34 + bbits));
    unsigned long long h = 0;
    SG_CUDA(cudaMemcpy(&h, nz.p, sizeof(h), cudaMemcpyDeviceToHost));
    P.part.zlo = kind == 1 ? -1 : hi - (int64_t)h;
    k_px_invert<<<grid_n(nv), 256>>>(P.part.perm.p, nv, P.part.inv.p);
    SG_CUDA(cudaGetLastError());
  }
  auto scan_len = [&](const int64_t *off, int64_t rlo, int64_t rhi, DBuf<int64_t> &out) {
    DBuf<int64_t> len(nv + 1);
    k_px_len<<<grid_n(nv + 1), 256>>>(off, P.part.perm.p, nv, rlo, rhi, len.p);
    SG_CUDA(cudaGetLastError());
    out.alloc((size_t)nv + 1);
    size_t tb = 0;
    SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, out.p, (int)(nv + 1)));
    DBuf<char> t(std::max<size_t>(tb, 1));
    SG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, len.p, out.p, (int)(nv + 1)));
  };
  auto view = std::make_unique<View>();
  view->nv = nv;
  scan_len(v.off.p, lo, hi, view->off);
  int64_t ne = 0;
  SG_CUDA(cudaMemcpy(&ne, view->off.p + nv, sizeof(int64_t), cudaMemcpyDeviceToHost));
  view->ne = ne;
  view->col.alloc((size_t)std::max<int64_t>(ne, 1));
  const bool w = kind == 0 && g.weighted;
  if (w) {
    P.weighted = true;
    P.w64.alloc((size_t)std::max<int64_t>(ne, 1));
  }
  k_px_copy_rows<<<grid_n(std::max<int64_t>(hi - lo, 1) * 32), 256>>>(
      v.off.p, v.col.p, w ? g.w64.p : nullptr, P.part.perm.p, P.part.inv.p, lo, hi, view->off.p,
      view->col.p, w ? P.w64.p : nullptr);
  SG_CUDA(cudaGetLastError());
  SG_CUDA(cudaDeviceSynchronize());
  P.ne = ne;
  if (w) {
    weights_finalize(P);
    P.wmin = g.wmin, P.wmax = g.wmax;
    if (!g.w32.p) P.w32.release();
  }
  if (kind == 1) {  // pr: out-degrees of every vertex in the new numbering
    P.csr.nv = nv;
    scan_len(g.csr.off.p, 0, nv, P.csr.off);
    P.csc_ = std::move(view);
  } else {
    // push / symmetrized rows: ascending targets (min and count apps do not
    // depend on the order; pr's CSC keeps it -- it is the summation order)
    const bool f64path = w && (!P.w32.p || (double)P.wmax * (double)std::max<int64_t>(nv - 1, 1) >= 4294967295.0);
    if (!f64path) sort_rows(*view, w && P.w32.p ? &P.w32 : nullptr);
    if (kind == 0) P.csr = std::move(*view);
    else P.sym_ = std::move(view);
  }
  SG_CUDA(cudaDeviceSynchronize());
}

std::unique_ptr<Graph> make_partition(Graph &g, int kind, int world, int rank, int relabel = 0) {
  if (g.is_part()) throw Error(SG_ECONFIG, "graph is already a partition");
  if (kind < 0 || kind > 2) throw Error(SG_ECONFIG, "partition kind must be 0 (CSR), 1 (CSC) or 2 (symmetrized)");
  if (world < 1 || world > kMaxParts || rank < 0 || rank >= world)
    throw Error(SG_ECONFIG, "bad rank / world size");
  if (g.nv > 0x7fffffffLL) throw Error(SG_ERANGE, "vertex ids must fit int32");
  const View &v = kind == 0 ? g.csr : kind == 1 ? g.csc() : g.sym();
  const Cuts c = make_cuts(v, world);
  auto P = std::make_unique<Graph>();
  P->nv = g.nv;
  P->part.kind = kind, P->part.rank = rank, P->part.world = world;
  P->part.cuts.assign(c.c, c.c + world + 1);
  P->part.lo = c.c[rank], P->part.hi = c.c[rank + 1];
  P->part.full_ne = v.ne;
  if (want_part_relabel(g, relabel)) {
    relabeled_slice(g, v, kind, c, *P);
    return P;
  }
  int64_t e0 = 0, e1 = 0;
  auto slice = std::make_unique<View>();
  slice_view(*slice, v, P->part.lo, P->part.hi, &e0, &e1);
  P->ne = slice->ne;
  if (kind == 0) {
    P->csr = std::move(*slice);
    if (g.weighted) {  // the rows' weights (graph.py:35-37), + the u32 kernel copy
      P->weighted = true;
      P->w64.alloc((size_t)std::max<int64_t>(P->ne, 1));
      if (P->ne)
        SG_CUDA(cudaMemcpy(P->w64.p, g.w64.p + e0, sizeof(int64_t) * P->ne,
                           cudaMemcpyDeviceToDevice));
      weights_finalize(*P);
      // every rank must pick the same label width: the full graph's bounds decide
      P->wmin = g.wmin, P->wmax = g.wmax;
      if (!g.w32.p) P->w32.release();
      if (g.w32.p && !P->w32.p) throw Error(SG_ECUDA, "partition weights: u32 copy missing");
    }
  } else {
    // pr divides by out-degrees of every vertex: keep the full CSR offsets
    if (kind == 1) {
      P->csr.nv = g.nv;
      P->csr.off.alloc((size_t)g.nv + 1);
      SG_CUDA(cudaMemcpy(P->csr.off.p, g.csr.off.p, sizeof(int64_t) * (g.nv + 1),
                         cudaMemcpyDeviceToDevice));
      P->csc_ = std::move(slice);
    } else {
      P->sym_ = std::move(slice);
    }
  }
  SG_CUDA(cudaDeviceSynchronize());
  return P;
}

// ----------------------------------------------------- ranks as threads --
void run_peer_threads(Graph &g, const sg_params &p, int world, const Out &o) {
  const int kind = part_kind_of(p.app);
  std::vector<std::unique_ptr<Graph>> parts;
  const int relabel = (p.flags & SG_FLAG_RELABEL) ? 1 : (p.flags & SG_FLAG_NO_RELABEL) ? -1 : 0;
  for (int r = 0; r < world; ++r) parts.push_back(make_partition(g, kind, world, r, relabel));
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev));
  std::vector<std::unique_ptr<Team>> teams;
  const Layout lay = Layout::of(g.nv);
  for (int r = 0; r < world; ++r) {
    auto T = std::make_unique<Team>();
    T->rank = r, T->world = world, T->device = dev, T->lay = lay;
    SG_CUDA(cudaMalloc(&T->base, lay.bytes));
    SG_CUDA(cudaMemset(T->base, 0, sizeof(Hdr)));
    teams.push_back(std::move(T));
  }
  HostBarrier hb(world);
  for (auto &T : teams) {
    for (int q = 0; q < world; ++q) T->peer[q] = teams[(size_t)q]->base;
    T->connected = true;
    T->host = &hb;
  }
  preload_peer_kernels();
  SG_CUDA(cudaDeviceSynchronize());
  std::vector<std::string> err(world);
  std::vector<int> code(world, SG_OK);
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      try {
        SG_CUDA(cudaSetDevice(dev));
        std::vector<sg_round> rr(r == 0 ? 0 : 1);
        std::vector<double> lab(r == 0 ? 0 : (size_t)g.nv);
        int64_t nr = 0;
        double ms = 0;
        Out ro = r == 0 ? o : Out{lab.data(), nullptr, 0, &nr, &ms};
        team_run(*teams[(size_t)r], *parts[(size_t)r], p, ro);
      } catch (const Error &e) {
        err[r] = e.what(), code[r] = e.code;
        hb.fail();
      } catch (const std::exception &e) {
        err[r] = e.what(), code[r] = SG_ECUDA;
        hb.fail();
      }
    });
  for (auto &t : th) t.join();
  SG_CUDA(cudaDeviceSynchronize());
  for (int r = 0; r < world; ++r)  // the first real failure (not "a peer rank failed")
    if (code[r] != SG_OK && err[r] != "a peer rank failed") throw Error(code[r], err[r]);
  for (int r = 0; r < world; ++r)
    if (code[r] != SG_OK) throw Error(code[r], err[r]);
}

}  // namespace
}  // namespace sg

struct sg_team {
  std::unique_ptr<sg::Team> t;
};

using sg::Error;

extern "C" {

int sg_graph_partition(sg_graph *gh, int32_t kind, int32_t world, int32_t rank, sg_graph **out) {
  return sg::guard([&] {
    if (!gh || !out) throw Error(SG_ECONFIG, "null argument");
    const int relabel = (kind & SG_PART_RELABEL) ? 1 : (kind & SG_PART_NO_RELABEL) ? -1 : 0;
    auto P = sg::make_partition(*gh->g, kind & 0xff, world, rank, relabel);
    *out = new sg_graph{std::shared_ptr<sg::Graph>(P.release())};
  });
}

int sg_graph_part_info(sg_graph *gh, int32_t *kind, int32_t *rank, int32_t *world,
                       int64_t *cuts_out, int64_t *full_ne) {
  return sg::guard([&] {
    const sg::Graph &g = *gh->g;
    if (kind) *kind = g.part.kind;
    if (rank) *rank = g.part.rank;
    if (world) *world = g.part.world;
    if (cuts_out && g.is_part())
      for (size_t i = 0; i < g.part.cuts.size(); ++i) cuts_out[i] = g.part.cuts[i];
    if (full_ne) *full_ne = g.part.full_ne;
  });
}

int sg_team_create(int32_t rank, int32_t world, int64_t nv, sg_team **out, uint8_t handle_out[64]) {
  return sg::guard([&] {
    if (world < 1 || world > sg::kMaxParts || rank < 0 || rank >= world)
      throw Error(SG_ECONFIG, "bad rank / world size");
    if (nv < 0 || nv > 0x7fffffffLL) throw Error(SG_ERANGE, "vertex count out of range");
    auto T = std::make_unique<sg::Team>();
    T->rank = rank, T->world = world, T->lay = sg::Layout::of(nv);
    SG_CUDA(cudaGetDevice(&T->device));
    SG_CUDA(cudaMalloc(&T->base, T->lay.bytes));
    SG_CUDA(cudaMemset(T->base, 0, sizeof(sg::Hdr)));
    SG_CUDA(cudaDeviceSynchronize());
    T->peer[rank] = T->base;
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t size");
    cudaIpcMemHandle_t h;
    SG_CUDA(cudaIpcGetMemHandle(&h, T->base));
    std::memcpy(handle_out, &h, 64);
    if (world == 1) T->connected = true;
    *out = new sg_team{std::move(T)};
  });
}

int sg_team_connect(sg_team *tm, const uint8_t *handles) {
  return sg::guard([&] {
    sg::Team &T = *tm->t;
    if (T.connected) return;
    for (int q = 0; q < T.world; ++q) {
      if (q == T.rank) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * (size_t)q, 64);
      void *p = nullptr;
      SG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      T.peer[q] = static_cast<char *>(p);
      T.ipc[q] = true;
    }
    T.connected = true;
  });
}

int sg_team_run(sg_team *tm, sg_graph *gh, const sg_params *p, double *labels_out,
                sg_round *rounds_out, int64_t rounds_cap, int64_t *nrounds, double *ms_out) {
  return sg::guard([&] {
    if (!tm || !gh || !p || !nrounds) throw Error(SG_ECONFIG, "null argument");
    sg::team_run(*tm->t, *gh->g, *p, sg::Out{labels_out, rounds_out, rounds_cap, nrounds, ms_out});
  });
}

void sg_team_destroy(sg_team *tm) { delete tm; }

int sg_peer_run_threads(sg_graph *gh, const sg_params *p, int32_t world, double *labels_out,
                        sg_round *rounds_out, int64_t rounds_cap, int64_t *nrounds,
                        double *ms_out) {
  return sg::guard([&] {
    if (world < 1 || world > sg::kMaxParts) throw Error(SG_ECONFIG, "bad world size");
    if (p->devices != world) throw Error(SG_ECONFIG, "params.devices must equal world");
    sg::run_peer_threads(*gh->g, *p, world,
                         sg::Out{labels_out, rounds_out, rounds_cap, nrounds, ms_out});
  });
}

}  // extern "C"
