// sg_distk.cuh — per-round counter kernels shared by the edge-cut drivers
// (NCCL / ranks-as-threads: sg_dist.cu, sg_dist_push.cu; NVLink peer memory:
// sg_peer.cu).  A rank's counter block is summed over ranks (the transport's
// reduction) before the advance kernel writes the round log (engine.py:116-163,
// 205-235) and decides quiescence.
#pragma once
#include "sg_runtime.cuh"

namespace sg {
namespace {

constexpr int kDP = 12;  // counter block: fsize, edges, nhuge, huge_edges, nlarge,
                         // large_edges, sent, bcast, twc, lb, next, pad

__global__ void k_dp_collect(PushArgs a, long long *acc) {
  const Ctl *ctl = a.ctl;
  if (threadIdx.x || ctl->done) return;
  const long long fs = ctl->dense ? a.dense_n : ctl->fsize;
  acc[0] = fs;
  acc[1] = (long long)ctl->edges;
  acc[2] = a.sched >= 2 ? 0 : ctl->nhuge;
  acc[3] = a.sched >= 2 ? 0 : (long long)ctl->huge_edges;
  acc[4] = a.sched >= 2 ? 0 : ctl->nlarge;
  acc[5] = a.sched >= 2 ? 0 : (long long)ctl->large_edges;
  acc[8] = a.sched == 1 ? 0 : fs > 0;  // run_round only for a non-empty local frontier
  acc[9] = a.sched == 1 ? ctl->huge_edges > 0 : a.sched == 0 ? ctl->nhuge > 0 : 0;
}

__global__ void k_dp_advance(PushArgs a, long long *acc, Loop lp) {
  Ctl *ctl = a.ctl;
  if (threadIdx.x || ctl->done) return;
  const uint32_t round = ctl->round;
  RoundStat &s = a.stats[round];
  s.frontier_size = acc[0];
  s.active_edges = acc[1];
  s.huge_count = acc[2];
  s.huge_edges = acc[3];
  s.large_count = acc[4];
  s.large_edges = acc[5];
  s.updated = acc[10];
  s.comm_sent = acc[6];
  s.comm_broadcast = acc[7];
  s.launches_twc = acc[8];
  s.launches_lb = acc[9];
  ctl->fsize = ctl->nsize;
  ctl->nsize = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = ctl->chunk_head = 0;
  ctl->edges = ctl->huge_edges = ctl->large_edges = 0;
  ctl->dense = 0;
  ctl->round = round + 1;
  const bool empty = acc[10] == 0;
  for (int i = 0; i < kDP; ++i) acc[i] = 0;
  loop_test(ctl, round, empty, lp);
}

template <class T>
__global__ void k_iota_from(T *p, int64_t n, int64_t base) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    p[i] = (T)(base + i);
}

constexpr int kDistN = 12;  // counter block summed over ranks each round

// pr: {twc launches, lb launches, nhuge, huge_edges, nlarge, large_edges}
__global__ void k_dist_pr_collect(const Ctl *ctl, int has_rows, long long *acc) {
  if (threadIdx.x || ctl->done) return;
  acc[0] = has_rows;
  acc[1] = ctl->nhuge > 0;
  acc[2] = ctl->nhuge;
  acc[3] = (long long)ctl->huge_edges;
  acc[4] = ctl->nlarge;
  acc[5] = (long long)ctl->large_edges;
}

// kcore, after the count phase and the kill: this rank's round counters
__global__ void k_dist_kc_collect(PullArgs a, long long *acc) {
  const Ctl *ctl = a.ctl;
  if (threadIdx.x || ctl->done) return;
  // fzero: isolated rows killed at init (peer relabeled blocks), round 0 only
  const long long fs = ctl->dense ? (long long)a.row_n + ctl->fzero : ctl->fsize;
  acc[0] = fs;
  acc[1] = (long long)ctl->edges;
  acc[2] = ctl->nhuge;
  acc[3] = (long long)ctl->huge_edges;
  acc[4] = ctl->nlarge;
  acc[5] = (long long)ctl->large_edges;
  acc[6] = (long long)ctl->ndying + ctl->fzero;
  acc[7] = (long long)ctl->comm_bcast;
  acc[8] = fs > 0;            // run_round only for a non-empty local frontier (engine.py:216)
  acc[9] = ctl->nhuge > 0;
}

// owned vertices marked this round (alive neighbours of any rank's dying
// vertices, after the mark all-reduce) -> this rank's next local frontier
__global__ void k_dist_kc_compact(const Ctl *ctl, const uint32_t *mark, uint32_t lo, uint32_t hi,
                                  uint32_t *q0, uint32_t *q1, uint32_t *nsize) {
  if (ctl->done) return;
  const uint32_t round = ctl->round, stamp = round + 1;
  uint32_t *q = (round & 1) ? q0 : q1;
  const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < hi - lo; b += st) {
    const uint64_t i = b + threadIdx.x;
    const bool m = i < hi - lo && mark[lo + i] == stamp;
    warp_append(m, lo + (uint32_t)i, q, nsize);
  }
}

__global__ void k_dist_kc_next(const Ctl *ctl, long long *acc) {
  if (threadIdx.x || ctl->done) return;
  acc[10] = ctl->nsize;
}

// kcore round bookkeeping from the rank-summed counters (apps.py:220-232)
__global__ void k_dist_kc_advance(PullArgs a, long long *acc, Loop lp) {
  Ctl *ctl = a.ctl;
  if (threadIdx.x || ctl->done) return;
  const uint32_t round = ctl->round;
  RoundStat &s = a.stats[round];
  s.frontier_size = acc[0];
  s.active_edges = acc[1];
  s.huge_count = acc[2];
  s.huge_edges = acc[3];
  s.large_count = acc[4];
  s.large_edges = acc[5];
  s.updated = acc[6];
  s.comm_sent = 0;
  s.comm_broadcast = acc[7];
  s.launches_twc = acc[8];
  s.launches_lb = acc[9];
  const bool stop = acc[6] == 0 || acc[10] == 0;
  ctl->fsize = ctl->nsize;
  ctl->nsize = 0;
  ctl->ndying = ctl->fzero = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = ctl->chunk_head = 0;
  ctl->edges = ctl->huge_edges = ctl->large_edges = ctl->comm_bcast = 0;
  ctl->dense = 0;
  ctl->round = round + 1;
  for (int i = 0; i < kDistN; ++i) acc[i] = 0;
  loop_test(ctl, round, stop, lp);
}

}  // namespace
}  // namespace sg
