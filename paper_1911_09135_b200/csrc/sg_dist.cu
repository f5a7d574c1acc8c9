// sg_dist.cu — edge-cut partitioned BSP for the push apps (bfs / sssp / cc).
//
// Reference: make_partition / sync_labels / the per-device loop of
// engine.py:64-113, 184-235.  Partition d owns the contiguous, edge-balanced
// row block [c[d], c[d+1]) of the traversal view and keeps a full-length label
// copy.  One BSP round:
//   1. every partition runs the ALB round (inspection, huge LB kernel, TWC
//      bins) over its LOCAL frontier, lowering its own label copy;
//   2. exchange: merged = min over partitions of their next-half labels
//      (sync_labels with 'min'); comm_sent counts (partition, non-owned v)
//      pairs whose local copy dropped below the round-start snapshot
//      (out_d != baseline, engine.py:105-109);
//   3. diff: every changed vertex joins its OWNER's next local frontier;
//      comm_broadcast += mirror_count[v] (engine.py:232-234);
//   4. quiescence when no partition has a next frontier.
// Two communicators implement step 2-3:
//   * local — D partitions on this GPU (engine.run(devices=D); all arrays in
//     one HBM), a single exchange kernel; the whole loop is one CUDA-graph
//     WHILE launch, exactly like the single-partition engine;
//   * NCCL — one partition per rank / GPU (torchrun): ncclAllReduce(min) of
//     the label pairs over NVLink, a per-rank diff kernel over the owned
//     range, and ncclAllReduce(sum) of the round counters (quiescence).
//     libnccl is dlopen'ed (preferring the copy torch already loaded), so the
//     single-GPU library has no NCCL dependency.
// bfs runs as unit-weight relaxation (OpPair<1>): identical labels and rounds.
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "sg_comm.cuh"
#include "sg_prx.cuh"
#include "sg_distk.cuh"

namespace sg {
namespace {

// per-round counters summed over partitions (and over ranks with NCCL)
struct PartAcc {
  long long fsize, edges, nhuge, huge_edges, nlarge, large_edges, sent, bcast, twc, lb, next;
};
constexpr int kAccN = sizeof(PartAcc) / sizeof(long long);

template <class L>
struct PartLabs {
  L *p[kMaxParts];
};
struct PartCtl {
  Ctl *ctl[kMaxParts];
  uint32_t *q[kMaxParts][2];
};

// a partition finished its round kernels: fold its counters, reset them
__global__ void k_part_collect(Ctl *pc, uint32_t dense_n, PartAcc *acc) {
  if (threadIdx.x || pc->done) return;
  const long long fs = pc->dense ? dense_n : pc->fsize;
  acc->fsize += fs;
  acc->edges += (long long)pc->edges;
  acc->nhuge += pc->nhuge;
  acc->huge_edges += (long long)pc->huge_edges;
  acc->nlarge += pc->nlarge;
  acc->large_edges += (long long)pc->large_edges;
  acc->twc += fs > 0;         // run_round only for a non-empty local frontier (engine.py:216)
  acc->lb += pc->nhuge > 0;   // lb launch only if the inspection found huge vertices
  pc->edges = pc->huge_edges = pc->large_edges = 0;
  pc->nhuge = pc->nlarge = pc->large_head = pc->chunk_head = 0;
  pc->nsize = 0;
}

// group lanes by owner partition and append the changed vertices of each group
__device__ __forceinline__ void append_by_owner(bool changed, int own, uint32_t v,
                                                const PartCtl &pc, uint32_t round) {
  const uint32_t grp = __match_any_sync(kFull, changed ? own : -1);
  if (!changed) return;
  const int leader = __ffs(grp) - 1;
  uint32_t base = 0;
  Ctl *c = pc.ctl[own];
  if ((int)lane_id() == leader) base = atomicAdd(&c->nsize, (uint32_t)__popc(grp));
  base = __shfl_sync(grp, base, leader);
  uint32_t *q = (round & 1) ? pc.q[own][0] : pc.q[own][1];  // next frontier of round+1
  q[base + __popc(grp & lanemask_lt())] = v;
}

// local communicator: exchange + diff for D partitions held on this GPU
template <class L>
__global__ void __launch_bounds__(256) k_exchange_local(PartLabs<L> labs, int D, int64_t nv,
                                                        Cuts cuts, PartCtl pc,
                                                        const uint32_t *mc, const Ctl *g,
                                                        PartAcc *acc) {
  __shared__ unsigned long long red[32];
  if (g->done) return;
  const uint32_t round = g->round, ch = round & 1u, nh = ch ^ 1u;
  unsigned long long sent = 0, bc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < nv; b += stride) {
    const int64_t v = b + threadIdx.x;
    bool changed = false;
    int own = 0;
    if (v < nv) {
      own = owner_of(cuts, (uint32_t)v);
      const L cur = labs.p[0][2 * v + ch];
      L m = cur;
      for (int d = 0; d < D; ++d) {
        const L x = labs.p[d][2 * v + nh];
        sent += (x < cur && d != own);  // a stale next half is >= cur, never counted
        m = x < m ? x : m;
      }
      for (int d = 0; d < D; ++d) labs.p[d][2 * v + nh] = m;
      changed = m < cur;
      if (changed) bc += mc[v];
    }
    append_by_owner(changed, own, (uint32_t)v, pc, round);
  }
  unsigned long long s = block_sum(sent, red);
  if (threadIdx.x == 0 && s) atomicAdd((unsigned long long *)&acc->sent, s);
  s = block_sum(bc, red);
  if (threadIdx.x == 0 && s) atomicAdd((unsigned long long *)&acc->bcast, s);
}

// NCCL communicator, before the all-reduce: this rank's sent count
template <class L>
__global__ void __launch_bounds__(256) k_count_sent(const L *lab, int64_t nv, long long lo,
                                                    long long hi, const Ctl *g, PartAcc *acc) {
  __shared__ unsigned long long red[32];
  if (g->done) return;
  const uint32_t ch = g->round & 1u, nh = ch ^ 1u;
  unsigned long long sent = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride)
    if ((v < lo || v >= hi) && lab[2 * v + nh] < lab[2 * v + ch]) ++sent;
  sent = block_sum(sent, red);
  if (threadIdx.x == 0 && sent) atomicAdd((unsigned long long *)&acc->sent, sent);
}

// NCCL communicator, after the all-reduce: owned changed vertices -> next frontier
template <class L>
__global__ void __launch_bounds__(256) k_diff_owned(const L *lab, long long lo, long long hi,
                                                    PartCtl pc, const uint32_t *mc, const Ctl *g,
                                                    PartAcc *acc) {
  __shared__ unsigned long long red[32];
  if (g->done) return;
  const uint32_t round = g->round, ch = round & 1u, nh = ch ^ 1u;
  unsigned long long bc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = lo + (int64_t)blockIdx.x * blockDim.x; b < hi; b += stride) {
    const int64_t v = b + threadIdx.x;
    bool changed = false;
    if (v < hi) {
      changed = lab[2 * v + nh] < lab[2 * v + ch];
      if (changed) bc += mc[v];
    }
    append_by_owner(changed, 0, (uint32_t)v, pc, round);
  }
  bc = block_sum(bc, red);
  if (threadIdx.x == 0 && bc) atomicAdd((unsigned long long *)&acc->bcast, bc);
}

__global__ void k_acc_next(PartCtl pc, int D, const Ctl *g, PartAcc *acc) {
  if (threadIdx.x || g->done) return;
  for (int d = 0; d < D; ++d) acc->next += pc.ctl[d]->nsize;
}

// global round bookkeeping + loop test (sets every partition's done flag)
__global__ void k_part_advance(PartCtl pc, int D, Ctl *g, PartAcc *acc, RoundStat *stats,
                               Loop lp) {
  if (threadIdx.x) return;
  if (g->done) {
    if (lp.use_cond) cudaGraphSetConditional(lp.cond, 0u);
    return;
  }
  const uint32_t r = g->round;
  RoundStat &s = stats[r];
  s.frontier_size = acc->fsize;
  s.active_edges = acc->edges;
  s.huge_count = acc->nhuge;
  s.huge_edges = acc->huge_edges;
  s.large_count = acc->nlarge;
  s.large_edges = acc->large_edges;
  s.updated = acc->next;
  s.comm_sent = acc->sent;
  s.comm_broadcast = acc->bcast;
  s.launches_twc = acc->twc;
  s.launches_lb = acc->lb;
  const bool empty = acc->next == 0;
  *acc = PartAcc{};
  g->round = r + 1;
  loop_test(g, r, empty, lp);
  for (int d = 0; d < D; ++d) {
    Ctl *c = pc.ctl[d];
    c->fsize = c->nsize;
    c->nsize = 0;
    c->dense = 0;
    c->round = r + 1;
    c->done = g->done;
  }
}

// -------------------------------------------------------------- the driver
struct PartRunner {
  Graph &g;
  const sg_params &p;
  const View *v = nullptr;
  int64_t nv = 0, thr = 0, max_rounds = 0;
  Cuts cuts{};
  int first = 0, nlocal = 0;  // partitions executed by this process
  std::vector<RunBufs> rb;
  DBuf<Ctl> gctl;
  DBuf<PartAcc> acc;
  DBuf<RoundStat> stats;
  int64_t stats_cap = 0;
  DBuf<uint32_t> mc;
  std::vector<std::shared_ptr<void>> keep;

  PartRunner(Graph &g_, const sg_params &p_, int64_t thr_, int64_t max_rounds_, int D, int first_,
             int nlocal_)
      : g(g_), p(p_), thr(thr_), max_rounds(max_rounds_), first(first_), nlocal(nlocal_) {
    v = p.app == SG_APP_CC ? &g.sym() : &g.csr;
    nv = v->nv;
    cuts = make_cuts(*v, D);
    mc.alloc(std::max<int64_t>(nv, 1));
    mirror_counts(*v, cuts, mc.p);
    rb.resize(nlocal);
    stats_cap = ::sg::stats_cap(max_rounds);
    for (int i = 0; i < nlocal; ++i) rb[i].alloc_common(nv, 1);
    gctl.alloc(1);
    acc.alloc(1);
    stats.alloc(stats_cap);
  }
  PushArgs args(int i) {
    const int d = first + i;
    PushArgs a = rb[i].push_args(*v, thr);
    a.no_enqueue = 1;
    a.dense_lo = (uint32_t)cuts.c[d];
    a.dense_n = (uint32_t)(cuts.c[d + 1] - cuts.c[d]);
    return a;
  }
  PartCtl part_ctl() {
    PartCtl pc{};
    for (int i = 0; i < nlocal; ++i) {
      pc.ctl[i] = rb[i].ctl.p;
      pc.q[i][0] = rb[i].q0.p;
      pc.q[i][1] = rb[i].q1.p;
    }
    return pc;
  }
  // initial local frontiers (apps.py:94-95, 126-127) + control blocks
  void init(cudaStream_t s) {
    const bool cc = p.app == SG_APP_CC;
    for (int i = 0; i < nlocal; ++i) {
      const int d = first + i;
      const bool owns_src = p.source >= cuts.c[d] && p.source < cuts.c[d + 1];
      const uint32_t n0 = cc ? (uint32_t)(cuts.c[d + 1] - cuts.c[d]) : (owns_src ? 1u : 0u);
      k_ctl_init<<<1, 1, 0, s>>>(rb[i].ctl.p, (int32_t)cc, n0);
      if (!cc && owns_src) k_set1<uint32_t><<<1, 1, 0, s>>>(rb[i].q0.p, 0, (uint32_t)p.source);
    }
    k_ctl_init<<<1, 1, 0, s>>>(gctl.p, 0, 0);
    SG_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(PartAcc), s));
    SG_CUDA(cudaGetLastError());
  }
};

template <class L>
void init_pairs(L *lab, int64_t nv, bool cc, int64_t src, cudaStream_t s) {
  if (cc) {
    k_iota_pairs<<<grid_n(nv), 256, 0, s>>>((uint32_t *)lab, nv);
  } else {
    const L inf = sizeof(L) == 4 ? (L)kInf32 : (L)0x7ff0000000000000ull;
    k_fill<L><<<grid_n(2 * nv), 256, 0, s>>>(lab, 2 * nv, inf);
    k_set1<L><<<1, 1, 0, s>>>(lab, 2 * src, (L)0);
    k_set1<L><<<1, 1, 0, s>>>(lab, 2 * src + 1, (L)0);
  }
  SG_CUDA(cudaGetLastError());
}

template <class L, class Op>
void run_partitioned(PartRunner &R, const std::vector<L *> &labs, const std::vector<Op> &ops,
                     Comm *comm, double *labels_out, sg_round *rounds_out, int64_t cap,
                     int64_t *nrounds, double *ms_out) {
  const bool blocked = R.p.blocked != 0;
  const int D = R.cuts.D;
  const int64_t nv = R.nv;
  PartLabs<L> pl{};
  for (int i = 0; i < R.nlocal; ++i) pl.p[i] = labs[i];
  const PartCtl pc = R.part_ctl();
  Ctl *g = R.gctl.p;
  PartAcc *acc = R.acc.p;
  const uint32_t *mc = R.mc.p;
  const int64_t limit = std::min<int64_t>(R.max_rounds, R.stats_cap);

  auto partition_rounds = [&](RoundCtx &c) {
    for (int i = 0; i < R.nlocal; ++i) {
      const PushArgs a = R.args(i);
      push_round(c, a, ops[i], blocked);
      c.L.go("part_collect", k_part_collect, 1, 32, c.s, a.ctl, a.dense_n, acc);
    }
  };
  cudaStream_t s;
  SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  SG_CUDA(cudaEventCreate(&e0));
  SG_CUDA(cudaEventCreate(&e1));
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  Launcher lau;
  auto cleanup = [&] {
    cudaStreamSynchronize(s);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
  };
  try {
    size_t body_nodes = 0;
    if (!comm) {  // local: WHILE { partition rounds; exchange; advance }
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
      cudaGraph_t body = np.conditional.phGraph_out[0];
      SG_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
      RoundCtx c{lau, s, cond, 1};
      partition_rounds(c);
      lau.go("exchange", k_exchange_local<L>, grid_n(nv), 256, s, pl, D, nv, R.cuts, pc, mc,
           (const Ctl *)g, acc);
      lau.go("acc_next", k_acc_next, 1, 32, s, pc, R.nlocal, (const Ctl *)g, acc);
      lau.go("part_advance", k_part_advance, 1, 32, s, pc, R.nlocal, g, acc, R.stats.p,
           Loop{limit, R.max_rounds, cond, 1});
      SG_CUDA(cudaStreamEndCapture(s, &body));
      SG_CUDA(cudaGraphGetNodes(body, nullptr, &body_nodes));
      SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    }
    SG_CUDA(cudaEventRecord(e0, s));
    R.init(s);
    for (int i = 0; i < R.nlocal; ++i)
      init_pairs<L>(labs[i], nv, R.p.app == SG_APP_CC, R.p.source, s);
    if (!comm) {
      SG_CUDA(cudaGraphLaunch(exec, s));
    } else {  // NCCL: host-driven rounds (one partition on this rank)
      const long long lo = R.cuts.c[R.first], hi = R.cuts.c[R.first + 1];
      const CType dt = sizeof(L) == 4 ? CType::U32 : CType::U64;
      Ctl h;
      for (int64_t r = 0; r < limit + 1; ++r) {
        RoundCtx c{lau, s, cudaGraphConditionalHandle{}, 0};
        partition_rounds(c);
        lau.go("count_sent", k_count_sent<L>, grid_n(nv), 256, s, (const L *)labs[0], nv, lo, hi,
             (const Ctl *)g, acc);
        comm->allreduce(labs[0], 2 * nv, dt, COp::Min, s);
        lau.go("diff", k_diff_owned<L>, grid_n(hi - lo), 256, s, (const L *)labs[0], lo, hi, pc, mc,
             (const Ctl *)g, acc);
        lau.go("acc_next", k_acc_next, 1, 32, s, pc, 1, (const Ctl *)g, acc);
        comm->allreduce(acc, kAccN, CType::I64, COp::Sum, s);
        lau.go("part_advance", k_part_advance, 1, 32, s, pc, 1, g, acc, R.stats.p,
             Loop{limit, R.max_rounds, cudaGraphConditionalHandle{}, 0});
        SG_CUDA(cudaMemcpyAsync(&h, g, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
        SG_CUDA(cudaStreamSynchronize(s));
        if (h.done) break;
      }
    }
    SG_CUDA(cudaEventRecord(e1, s));
    SG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms_out) *ms_out = ms;
    Ctl h;
    SG_CUDA(cudaMemcpy(&h, g, sizeof(Ctl), cudaMemcpyDeviceToHost));
    const int64_t rounds = h.round;
    g_launches.fetch_add((int64_t)body_nodes * rounds, std::memory_order_relaxed);
    std::vector<RoundStat> st((size_t)std::min<int64_t>(rounds, R.stats_cap));
    if (!st.empty())
      SG_CUDA(cudaMemcpy(st.data(), R.stats.p, sizeof(RoundStat) * st.size(),
                         cudaMemcpyDeviceToHost));
    if (rounds_out && !st.empty())
      std::memcpy(rounds_out, st.data(),
                  sizeof(RoundStat) * (size_t)std::min<int64_t>(cap, (int64_t)st.size()));
    *nrounds = rounds;
    if (labels_out) {
      DBuf<double> out(std::max<int64_t>(nv, 1));
      if (sizeof(L) == 4)
        k_labels_pair_u32<<<grid_n(nv), 256, 0, s>>>((const uint32_t *)labs[0], nv, g, out.p);
      else
        k_labels_pair_f64<<<grid_n(nv), 256, 0, s>>>((const unsigned long long *)labs[0], nv, g,
                                                     out.p);
      SG_CUDA(cudaGetLastError());
      SG_CUDA(cudaStreamSynchronize(s));
      SG_CUDA(cudaMemcpy(labels_out, out.p, sizeof(double) * nv, cudaMemcpyDeviceToHost));
    }
    if (h.error == SG_ECONVERGE)
      throw Error(SG_ECONVERGE,
                  "did not converge within " + std::to_string(R.max_rounds) + " rounds");
    if (h.error) throw Error(h.error, "round log capacity exhausted");
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

template <class L, class MakeOp>
void run_push_partitioned(PartRunner &R, MakeOp make_op, Comm *comm, double *labels_out,
                          sg_round *rounds_out, int64_t cap, int64_t *nrounds, double *ms_out) {
  std::vector<L *> labs;
  std::vector<decltype(make_op((L *)nullptr))> ops;
  for (int i = 0; i < R.nlocal; ++i) {
    auto b = std::make_shared<DBuf<L>>(2 * std::max<int64_t>(R.nv, 1));
    R.keep.push_back(b);
    labs.push_back(b->p);
    ops.push_back(make_op(b->p));
  }
  run_partitioned<L>(R, labs, ops, comm, labels_out, rounds_out, cap, nrounds, ms_out);
}

void dispatch_push(PartRunner &R, Comm *comm, double *labels_out, sg_round *rounds_out,
                   int64_t cap, int64_t *nrounds, double *ms_out) {
  Graph &g = R.g;
  const sg_params &p = R.p;
  if (p.app == SG_APP_CC)
    return run_push_partitioned<uint32_t>(
        R, [](uint32_t *l) { return OpPair<0>{l, nullptr, nullptr}; }, comm, labels_out,
        rounds_out, cap, nrounds, ms_out);
  const bool weighted = p.app == SG_APP_SSSP && g.weighted;
  if (!weighted)  // bfs == unit-weight relaxation (same labels and rounds)
    return run_push_partitioned<uint32_t>(
        R, [](uint32_t *l) { return OpPair<1>{l, nullptr, nullptr}; }, comm, labels_out,
        rounds_out, cap, nrounds, ms_out);
  const double bound = (double)g.wmax * (double)std::max<int64_t>(R.nv - 1, 1);
  if (g.w32.p && bound < 4294967295.0) {
    const uint32_t *w = g.w32.p;
    return run_push_partitioned<uint32_t>(
        R, [w](uint32_t *l) { return OpPair<2>{l, w, nullptr}; }, comm, labels_out, rounds_out,
        cap, nrounds, ms_out);
  }
  const int64_t *w = g.w64.p;
  return run_push_partitioned<unsigned long long>(
      R, [w](unsigned long long *l) { return OpPair<3>{l, nullptr, w}; }, comm, labels_out,
      rounds_out, cap, nrounds, ms_out);
}


// ------------------------------------------- pull apps, one partition per rank
// Reference: the pull view's row blocks (engine.py:64-85); a pull round writes
// only owned rows, so comm_sent is 0 and every changed value is broadcast to
// its mirrors (comm_broadcast, engine.py:232-234).
// pr over NCCL: this rank folds its edge-cut rows [lo, hi) with the exact-order
// pull (sg_prx.cuh, on a layout of its own rows), then every rank's new aux
// slice is broadcast, max |delta|, comm_broadcast and the bin counters are
// all-reduced, and the stop test runs on the reduced values.  eps_stop's gain
// is the maximum over ranks of the exact row sums of their own rows.
void run_pr_dist(Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds, Comm &cm,
                 double *labels_out, sg_round *rounds_out, int64_t cap, int64_t *nrounds,
                 double *ms_out) {
  const View &v = g.csc();
  const int64_t nv = v.nv;
  const Cuts cuts = make_cuts(v, cm.world);
  const uint32_t lo = (uint32_t)cuts.c[cm.rank], hi = (uint32_t)cuts.c[cm.rank + 1];
  RunBufs rb;
  rb.alloc_common(nv, stats_cap(max_rounds));
  PullArgs a = rb.pull_args(v, thr, 0);
  a.row_lo = lo, a.row_n = hi - lo;
  DBuf<uint32_t> mc;
  if (cm.world > 1) {
    mc.alloc(nv);
    mirror_counts(v, cuts, mc.p);
    a.mcount = mc.p;
  }
  DBuf<double> inv(nv), aux0(nv), aux1(nv), hacc(1), rank(nv);
  DBuf<unsigned long long> gmax(1);
  DBuf<long long> acc(kDistN);
  DBuf<uint32_t> head(1);
  const double d = p.damping, omd = 1.0 - p.damping;
  PrOp op{aux0.p, aux1.p, aux1.p, aux0.p, rank.p, inv.p, d, omd};
  op.mcount = a.mcount;
  PrFold fold{aux0.p, aux1.p, aux1.p, aux0.p, rank.p, inv.p, d, omd, a.mcount};
  Cuts one{};
  one.D = 1, one.c[0] = 0, one.c[1] = nv;
  Ctl *ctl = rb.ctl.p;
  const int64_t hs = exact_hs();
  const ExactLayout &XL = g.exact(hs, lo, hi);
  std::vector<std::unique_ptr<DBuf<char>>> keep;
  PrxArgs xa = prx_args(v, XL, std::max<int64_t>(thr, hs), thr != kNoHuge, ctl, nullptr, gmax.p,
                        head.p, [&](size_t bytes) {
                          keep.emplace_back(new DBuf<char>(bytes));
                          return (void *)keep.back()->p;
                        });
  const int gx = occupancy_grid(k_prx<0>, kTB);
  DistLoop dl;
  cudaStream_t s = dl.s;
  Launcher L;
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  PrStop st2{gmax.p, d, p.tol, v.ne, limit, max_rounds, cudaGraphConditionalHandle{}, 0, 1, 2,
             acc.p};
  SG_CUDA(cudaEventRecord(dl.e0, s));
  L.go("init", k_ctl_init, 1, 1, s, ctl, 1, (uint32_t)nv);
  L.go("init", k_pr_init, grid_n(nv), 256, s, g.csr.off.p, nv, omd, inv.p, rank.p, aux0.p);
  L.go("init", k_copy_f64, grid_n(nv), 256, s, (const double *)aux0.p, nv, aux1.p);
  fill<unsigned long long>(L, gmax.p, 1, 0ull, s);
  fill<long long>(L, acc.p, kDistN, 0ll, s);
  fill<uint32_t>(L, head.p, 1, 0u, s);
  fill<uint32_t>(L, xa.ck_meta, xa.nchunks, 0u, s);
  if (xa.nsplit) {
    L.go("init", k_prx_chunks, 1, 1024, s, xa.off, xa.big, xa.nsplit, (uint32_t *)xa.ck_first,
         (uint32_t *)xa.ck_row);
    L.go("pr_guess", k_prx_guess_sums, grid_n((int64_t)xa.nchunks * 32, kTB), kTB, s, xa,
         (const double *)inv.p);
    L.go("pr_guess", k_prx_guess_scan, grid_n((int64_t)xa.nsplit * 32, kTB), kTB, s, xa);
  }
  if (v.ne) {  // gain: exact sums of this rank's rows, then the max over ranks
    PrxArgs xg = xa;
    xg.gain = 1;
    L.go("pr_gain", k_prx<0>, gx, kTB, s, xg, fold);
    cm.allreduce(gmax.p, 1, CType::U64, COp::Max, s);
  }
  fill<uint32_t>(L, head.p, 1, 0u, s);
  if (xa.nsplit) {
    L.go("pr_guess", k_prx_guess_sums, grid_n((int64_t)xa.nchunks * 32, kTB), kTB, s, xa,
         (const double *)aux0.p);
    L.go("pr_guess", k_prx_guess_scan, grid_n((int64_t)xa.nsplit * 32, kTB), kTB, s, xa);
  }
  L.go("init", k_static_bins, grid_n(hi - lo), 256, s, v.off.p, lo, hi - lo, thr, rb.largeq.p,
       rb.hugeq.p, ctl, one);
  for (int64_t r = 0; r <= limit; ++r) {
    L.go("pr_pull", k_prx<0>, gx, kTB, s, xa, fold);
    L.go("dist", k_dist_pr_collect, 1, 32, s, (const Ctl *)ctl, (int)(hi > lo), acc.p);
    double *auxn = (r & 1) ? aux0.p : aux1.p;  // round r writes next1 / next0
    cm.group_begin();
    for (int q = 0; q < cm.world; ++q)
      cm.bcast(auxn + cuts.c[q], (size_t)(cuts.c[q + 1] - cuts.c[q]), CType::F64, q, s);
    cm.group_end();
    cm.allreduce(&ctl->delta_bits, 1, CType::U64, COp::Max, s);
    cm.allreduce(&ctl->comm_bcast, 1, CType::U64, COp::Sum, s);
    cm.allreduce(acc.p, 6, CType::I64, COp::Sum, s);
    L.go("pr_finish", k_pull_finish<PrOp, true>, 1, 1024, s, a, op, hacc.p, st2);
    fill<uint32_t>(L, head.p, 1, 0u, s);
    if (dl.done(ctl)) break;
  }
  cm.group_begin();  // every rank's rows -> the full label vector
  for (int q = 0; q < cm.world; ++q)
    cm.bcast(rank.p + cuts.c[q], (size_t)(cuts.c[q + 1] - cuts.c[q]), CType::F64, q, s);
  cm.group_end();
  SG_CUDA(cudaEventRecord(dl.e1, s));
  SG_CUDA(cudaEventSynchronize(dl.e1));
  float ms = 0;
  SG_CUDA(cudaEventElapsedTime(&ms, dl.e0, dl.e1));
  if (ms_out) *ms_out = ms;
  dist_results(rb, s, rank.p, nv, rounds_out, cap, nrounds, labels_out, max_rounds);
}

void run_kcore_dist(Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds, Comm &cm,
                    double *labels_out, sg_round *rounds_out, int64_t cap, int64_t *nrounds,
                    double *ms_out) {
  const bool classic = (p.flags & SG_FLAG_TWC_CLASSIC) != 0;
  const View &v = g.sym();
  const int64_t nv = v.nv;
  const Cuts cuts = make_cuts(v, cm.world);
  const uint32_t lo = (uint32_t)cuts.c[cm.rank], hi = (uint32_t)cuts.c[cm.rank + 1];
  RunBufs rb;
  rb.alloc_common(nv, stats_cap(max_rounds));
  rb.dying.alloc(std::max<int64_t>(nv, 1));
  PullArgs a = rb.pull_args(v, thr, 1);
  a.row_lo = lo, a.row_n = hi - lo;
  DBuf<uint32_t> mc;
  if (cm.world > 1) {
    mc.alloc(nv);
    mirror_counts(v, cuts, mc.p);
    a.mcount = mc.p;
  }
  PushArgs w = rb.push_args(v, kNoHuge);
  w.src_mode = 1;
  w.no_enqueue = 1;  // marks only; owners collect them after the exchange
  DBuf<uint8_t> alive(std::max<int64_t>(nv, 1));
  DBuf<uint32_t> mark(std::max<int64_t>(nv, 1)), hcnt(std::max<int64_t>(nv, 1));
  DBuf<double> labels(std::max<int64_t>(nv, 1));
  DBuf<long long> acc(kDistN);
  const KcOp op{alive.p, (uint32_t)std::min<int64_t>(p.k, 0xffffffffLL)};
  const OpMark mop{alive.p, mark.p};
  DistLoop dl;
  cudaStream_t s = dl.s;
  Launcher L;
  Ctl *ctl = rb.ctl.p;
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  const Loop lp{limit, max_rounds, cudaGraphConditionalHandle{}, 0};
  SG_CUDA(cudaEventRecord(dl.e0, s));
  L.go("init", k_ctl_init, 1, 1, s, ctl, 1, hi - lo);
  fill<uint8_t>(L, alive.p, nv, (uint8_t)1, s);
  fill<uint32_t>(L, mark.p, nv, 0u, s);
  fill<uint32_t>(L, hcnt.p, nv, 0u, s);
  fill<long long>(L, acc.p, kDistN, 0ll, s);
  for (int64_t r = 0; r <= limit; ++r) {
    RoundCtx c{L, s, cudaGraphConditionalHandle{}, 0};
    pull_round(c, a, op, p.blocked != 0, hcnt.p, classic);
    if (thr != kNoHuge)
      L.go("kcore_huge", k_pull_finish<KcOp, false>, 1, 1024, s, a, op, hcnt.p, PrStop{});
    L.go("kcore_kill", k_kcore_kill, grid_n(nv), 256, s, a, alive.p);
    L.go("dist", k_dist_kc_collect, 1, 32, s, a, acc.p);
    L.go("kcore_stats", k_kcore_reset, 1, 1, s, a);
    cm.allreduce(alive.p, nv, CType::U8, COp::Min, s);
    L.go("mark_twc", k_push_twc<OpMark>, occupancy_grid(k_push_twc<OpMark>, kTB), kTB, s, w, mop);
    L.go("mark_large", k_push_large<OpMark>, occupancy_grid(k_push_large<OpMark>, kTB), kTB, s,
         w, mop);
    cm.allreduce(mark.p, nv, CType::U32, COp::Max, s);
    L.go("dist", k_dist_kc_compact, grid_n(hi - lo), 256, s, (const Ctl *)ctl,
         (const uint32_t *)mark.p, lo, hi, rb.q0.p, rb.q1.p, &ctl->nsize);
    L.go("dist", k_dist_kc_next, 1, 32, s, (const Ctl *)ctl, acc.p);
    cm.allreduce(acc.p, kDistN, CType::I64, COp::Sum, s);
    L.go("advance", k_dist_kc_advance, 1, 32, s, a, acc.p, lp);
    if (dl.done(ctl)) break;
  }
  L.go("labels", k_labels_alive, grid_n(nv), 256, s, (const uint8_t *)alive.p, nv, labels.p);
  SG_CUDA(cudaEventRecord(dl.e1, s));
  SG_CUDA(cudaEventSynchronize(dl.e1));
  float ms = 0;
  SG_CUDA(cudaEventElapsedTime(&ms, dl.e0, dl.e1));
  if (ms_out) *ms_out = ms;
  dist_results(rb, s, labels.p, nv, rounds_out, cap, nrounds, labels_out, max_rounds);
}

// one rank of the edge-cut BSP over communicator `cm` (any app)
void dist_run_rank(Graph &g, const sg_params &p, Comm &cm, double *labels_out,
                   sg_round *rounds_out, int64_t cap, int64_t *nrounds, double *ms_out) {
  if (p.app < SG_APP_BFS || p.app > SG_APP_KCORE) throw Error(SG_ECONFIG, "unknown app");
  if ((p.app == SG_APP_BFS || p.app == SG_APP_SSSP) && (p.source < 0 || p.source >= g.nv))
    throw Error(SG_ECONFIG, "source " + std::to_string(p.source) + " outside graph");
  if (p.app == SG_APP_SSSP && g.weighted && g.wmin < 0)
    throw Error(SG_ECONFIG, "sssp requires non-negative weights");
  if (p.app == SG_APP_PR && !(p.damping > 0.0 && p.damping < 1.0))
    throw Error(SG_ECONFIG, "damping must be in (0, 1)");
  if (p.app == SG_APP_PR && !(p.tol > 0.0)) throw Error(SG_ECONFIG, "tolerance must be positive");
  if (p.app == SG_APP_KCORE && p.k < 1) throw Error(SG_ECONFIG, "k must be >= 1");
  const int64_t max_rounds =
      p.max_rounds > 0 ? p.max_rounds : 10 * std::max<int64_t>(g.nv, 1) + 256;
  if (p.sched < SG_SCHED_ALB || p.sched > SG_SCHED_EDGE) throw Error(SG_ECONFIG, "unknown scheduler");
  const int64_t thr = p.sched == SG_SCHED_TWC ? kNoHuge
                      : p.sched == SG_SCHED_ALB ? std::max<int64_t>(1, p.threshold)
                                                : 1;  // lb / vertex / edge: the LB path
  *nrounds = 0;
  if (ms_out) *ms_out = 0.0;
  if (g.nv == 0) return;
  if (p.app == SG_APP_PR) return run_pr_dist(g, p, thr, max_rounds, cm, labels_out, rounds_out, cap, nrounds, ms_out);
  if (p.app == SG_APP_KCORE) return run_kcore_dist(g, p, thr, max_rounds, cm, labels_out, rounds_out, cap, nrounds, ms_out);
  run_push_dist(g, p, thr, max_rounds, cm, labels_out, rounds_out, cap, nrounds, ms_out);
}

}  // namespace

// engine.run(devices=D > 1) for the push apps: D partitions on this GPU
void run_push_local_partitions(Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds,
                               double *labels_out, sg_round *rounds_out, int64_t cap,
                               int64_t *nrounds, double *ms_out) {
  PartRunner R(g, p, thr, max_rounds, p.devices, 0, p.devices);
  dispatch_push(R, nullptr, labels_out, rounds_out, cap, nrounds, ms_out);
}

}  // namespace sg

namespace sg {
namespace {
// One NCCL communicator per (unique id, rank, world), created on first use and
// reused by every later run: an ncclUniqueId bootstraps exactly one
// communicator (its root listener serves one init), and init costs far more
// than a BSP run.  Deliberately leaked at exit (destroying communicators after
// the CUDA runtime has torn down is unsafe); sg_nccl_release frees them.
// Entries are created OUTSIDE the map lock (ncclCommInitRank blocks until
// every rank of the id joined, and ranks driven from threads of one process
// must not serialise on it): a per-key slot with its own once-flag.  The key
// holds the device, so one id used on two devices gives two communicators.
struct CommSlot {
  std::once_flag once;
  std::unique_ptr<NcclComm> comm;
  std::exception_ptr err;
};
std::mutex g_comm_mu;
std::map<std::string, std::shared_ptr<CommSlot>> *g_comms =
    new std::map<std::string, std::shared_ptr<CommSlot>>();

void evict_comm(const std::string &key);

std::string comm_key(const uint8_t id[128], int rank, int world) {
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev));
  std::string key(reinterpret_cast<const char *>(id), 128);
  return key + ":" + std::to_string(rank) + "/" + std::to_string(world) + "@" + std::to_string(dev);
}

NcclComm &cached_comm(const std::string &key, const uint8_t id[128], int rank, int world) {
  std::shared_ptr<CommSlot> slot;
  {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto &p = (*g_comms)[key];
    if (!p) p = std::make_shared<CommSlot>();
    slot = p;
  }
  std::call_once(slot->once, [&] {
    try {
      slot->comm = std::make_unique<NcclComm>(id, rank, world);
    } catch (...) {
      slot->err = std::current_exception();
    }
  });
  if (slot->err) {
    evict_comm(key);
    std::rethrow_exception(slot->err);
  }
  return *slot->comm;
}

// a run that threw mid-collective leaves its communicator out of step with
// the peers: drop it so the next run with that id fails cleanly at init
void evict_comm(const std::string &key) {
  std::shared_ptr<CommSlot> old;
  std::lock_guard<std::mutex> lk(g_comm_mu);
  auto it = g_comms->find(key);
  if (it != g_comms->end()) old = it->second, g_comms->erase(it);
}
}  // namespace
}  // namespace sg

using sg::Error;

extern "C" {

int sg_nccl_unique_id(uint8_t id_out[128]) {
  return sg::guard([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    SG_NCCL(sg::nccl().getUniqueId(&id));
    std::memcpy(id_out, &id, 128);
  });
}


int sg_dist_run(sg_graph *gh, const sg_params *p, const uint8_t nccl_id[128], int32_t rank,
                int32_t world, double *labels_out, sg_round *rounds_out, int64_t rounds_cap,
                int64_t *nrounds, double *ms_out) {
  return sg::guard([&] {
    if (world < 1 || world > sg::kMaxParts || rank < 0 || rank >= world)
      throw Error(SG_ECONFIG, "bad rank / world size");
    const std::string key = sg::comm_key(nccl_id, rank, world);
    sg::NcclComm &comm = sg::cached_comm(key, nccl_id, rank, world);
    try {
      sg::dist_run_rank(*gh->g, *p, comm, labels_out, rounds_out, rounds_cap, nrounds, ms_out);
    } catch (...) {
      sg::evict_comm(key);
      throw;
    }
  });
}

void sg_nccl_release(void) {
  std::lock_guard<std::mutex> lk(sg::g_comm_mu);
  cudaDeviceSynchronize();
  sg::g_comms->clear();
}

int sg_dist_run_threads(sg_graph *gh, const sg_params *p, int32_t world, double *labels_out,
                        sg_round *rounds_out, int64_t rounds_cap, int64_t *nrounds,
                        double *ms_out) {
  return sg::guard([&] {
    if (world < 1 || world > sg::kMaxParts) throw Error(SG_ECONFIG, "bad world size");
    sg::Graph &g = *gh->g;
    if (p->app == SG_APP_CC || p->app == SG_APP_KCORE) g.sym();  // lazy views: build once
    if (p->app == SG_APP_PR) g.csc();
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    sg::ThreadHub hub(world);
    std::vector<std::string> err(world);
    std::vector<int> code(world, SG_OK);
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r)
      th.emplace_back([&, r] {
        try {
          SG_CUDA(cudaSetDevice(dev));
          sg::ThreadComm comm(hub, r);
          std::vector<sg_round> rr(r == 0 ? (size_t)std::max<int64_t>(rounds_cap, 0) : 0);
          std::vector<double> lab(r == 0 ? 0 : (size_t)g.nv);
          int64_t nr = 0;
          double ms = 0;
          sg::dist_run_rank(g, *p, comm, r == 0 ? labels_out : lab.data(),
                            r == 0 ? rounds_out : nullptr, r == 0 ? rounds_cap : 0, &nr, &ms);
          if (r == 0) {
            *nrounds = nr;
            if (ms_out) *ms_out = ms;
          }
        } catch (const Error &e) {
          err[r] = e.what(), code[r] = e.code;
          hub.fail();
        } catch (const std::exception &e) {
          err[r] = e.what(), code[r] = SG_ECUDA;
          hub.fail();
        }
      });
    for (auto &t : th) t.join();
    for (int r = 0; r < world; ++r)  // the first real failure (not "a peer rank failed")
      if (code[r] != SG_OK && err[r] != "a peer rank failed") throw Error(code[r], err[r]);
    for (int r = 0; r < world; ++r)
      if (code[r] != SG_OK) throw Error(code[r], err[r]);
  });
}

}  // extern "C"
