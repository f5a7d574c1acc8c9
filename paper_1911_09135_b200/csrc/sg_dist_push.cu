// sg_dist_push.cu — bfs / sssp / cc with one edge-cut partition per rank
// (engine.py:64-113, 205-235), on the single-device bitmap-frontier kernels.
//
// Every rank holds the whole graph view and a full label vector that is
// identical on all ranks at the start of a round; rank r owns rows [lo, hi).
// One BSP round:
//   1. relax: the ALB round (or lb / vertex / edge) over the LOCAL frontier
//      (changed owned vertices) lowers local labels anywhere and marks every
//      lowered vertex in the bitmap nb (red.min / red.or, sg_bm.cuh);
//   2. comm_sent = the marked vertices this rank does not own
//      (#{v not in own(d): out_d[v] != baseline}, engine.py:105-109) — exact,
//      because a mark is set iff the local copy went below the round start;
//   3. exchange (master / mirror, Gluon style), picked per round by volume:
//      * sparse: (id, label) of marked non-owned vertices go to their owners
//        (alltoallv), owners apply red.min; then every owner broadcasts the
//        (id, label) of its changed rows (alltoallv to all) — only updated
//        mirrors travel;
//      * dense: one all-reduce(min) of the label vector;
//   4. owners diff their rows against the round-start copy: changed rows form
//      the next local frontier (with their snapshot labels) and add their
//      mirror counts to comm_broadcast (engine.py:232-234);
//   5. counters are summed over ranks; the run ends when no rank has a
//      frontier (quiescence).
// bfs runs as unit-weight relaxation (identical labels and rounds).
#include "sg_comm.cuh"
#include "sg_distk.cuh"

namespace sg {
namespace {

// marked vertices owned by each rank (this rank's own rows excluded)
__global__ void __launch_bounds__(256) k_dp_count(const uint32_t *nb, int64_t nv, Cuts cuts,
                                                  int self, unsigned long long *cnt) {
  __shared__ unsigned int sc[kMaxParts];
  if (threadIdx.x < kMaxParts) sc[threadIdx.x] = 0;
  __syncthreads();
  const int64_t nw = (nv + 31) / 32, st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += st) {
    uint32_t x = nb[w];
    while (x) {
      const uint32_t v = (uint32_t)(w * 32) + (uint32_t)(__ffs(x) - 1);
      x &= x - 1;
      const int o = owner_of(cuts, v);
      if (o != self) atomicAdd(&sc[o], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x < cuts.D && sc[threadIdx.x]) atomicAdd(cnt + threadIdx.x, sc[threadIdx.x]);
}

// (id, label) of marked non-owned vertices, grouped by owner (cursor per owner)
template <class L>
__global__ void __launch_bounds__(256) k_dp_pack(const uint32_t *nb, const L *lab, int64_t nv,
                                                 Cuts cuts, int self,
                                                 unsigned long long *cursor, uint32_t *ids,
                                                 L *vals) {
  const int64_t nw = (nv + 31) / 32, st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += st) {
    uint32_t x = nb[w];
    while (x) {
      const uint32_t v = (uint32_t)(w * 32) + (uint32_t)(__ffs(x) - 1);
      x &= x - 1;
      const int o = owner_of(cuts, v);
      if (o == self) continue;
      const unsigned long long k = atomicAdd(cursor + o, 1ull);
      ids[k] = v;
      vals[k] = lab[v];
    }
  }
}

template <class L>
__global__ void k_dp_apply(const uint32_t *ids, const L *vals, int64_t n, L *lab) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    atomicMin(lab + ids[i], vals[i]);
}

// owner diff: changed rows -> next local frontier (+ snapshot), the update
// list for the mirrors, comm_broadcast; the round-start copy is advanced
template <class L>
__global__ void __launch_bounds__(256) k_dp_diff(const L *lab, L *own, uint32_t lo, uint32_t hi,
                                                 uint32_t *q, L *snap, Ctl *ctl,
                                                 const uint32_t *mc, uint32_t *uids, L *uvals,
                                                 long long *acc) {
  __shared__ unsigned long long red[32];
  if (ctl->done) return;
  unsigned long long bc = 0;
  const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < hi - lo; b += st) {
    const uint64_t i = b + threadIdx.x;
    bool ch = false;
    uint32_t v = 0;
    L x = 0;
    if (i < hi - lo) {
      v = lo + (uint32_t)i;
      x = lab[v];
      ch = x < own[i];
      if (ch) {
        own[i] = x;
        if (mc) bc += mc[v];
      }
    }
    const uint32_t slot = warp_append(ch, v, q, &ctl->nsize);
    if (ch) {
      snap[slot] = x;
      uids[slot] = v;
      uvals[slot] = x;
    }
  }
  bc = block_sum(bc, red);
  if (threadIdx.x == 0 && bc) atomicAdd((unsigned long long *)&acc[7], bc);
}

__global__ void k_dp_next(const Ctl *ctl, long long *acc, unsigned long long *sent) {
  if (threadIdx.x || ctl->done) return;
  acc[10] = ctl->nsize;
  acc[6] = (long long)*sent;
}

template <int KIND>
void run_dist_push(Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds, Comm &cm,
                   double *labels_out, sg_round *rounds_out, int64_t cap, int64_t *nrounds,
                   double *ms_out) {
  using Op = BmMin<KIND>;
  using L = typename Op::L;
  const CType LT = sizeof(L) == 4 ? CType::U32 : CType::U64;
  const bool cc = p.app == SG_APP_CC;
  const bool classic = (p.flags & SG_FLAG_TWC_CLASSIC) != 0;
  const View &v = cc ? g.sym() : g.csr;
  const int64_t nv = v.nv;
  const int D = cm.world, R = cm.rank;
  const Cuts cuts = make_cuts(v, D);
  const uint32_t lo = (uint32_t)cuts.c[R], hi = (uint32_t)cuts.c[R + 1];
  DBuf<uint32_t> mc;
  if (D > 1) {
    mc.alloc(nv);
    mirror_counts(v, cuts, mc.p);
  }
  RunBufs rb;
  rb.alloc_common(nv, stats_cap(max_rounds));
  PushArgs a = rb.push_args(v, thr);
  a.q[1] = a.q[0];
  a.dense_lo = lo, a.dense_n = hi - lo;
  a.sched = p.sched == SG_SCHED_LB ? 1 : p.sched == SG_SCHED_VERTEX ? 2 : p.sched == SG_SCHED_EDGE ? 3 : 0;
  const int64_t nw = (nv + 31) / 32 + 1;
  DBuf<L> lab(nv), snap(nv), own(std::max<int64_t>(hi - lo, 1)), uvals(nv), svals(nv), rvals(nv);
  DBuf<uint32_t> nb(nw), uids(nv), sids(nv), rids(nv);
  DBuf<long long> acc(kDP), tsum((nv + kFT - 1) / kFT + 1);
  DBuf<unsigned long long> cnt(kMaxParts + 1), cursor(kMaxParts);
  const bool weighted = p.app == SG_APP_SSSP && g.weighted;
  const Op op{lab.p, KIND == 2 ? g.w32.p : nullptr, KIND == 3 && weighted ? g.w64.p : nullptr,
              snap.p, nb.p};
  const bool owns_src = !cc && p.source >= lo && p.source < hi;
  const L inf = sizeof(L) == 4 ? (L)kInf32 : (L)0x7ff0000000000000ull;
  DistLoop dl;
  cudaStream_t s = dl.s;
  Launcher Lc;
  Ctl *ctl = rb.ctl.p;
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  const Loop lp{limit, max_rounds, cudaGraphConditionalHandle{}, 0};
  SG_CUDA(cudaEventRecord(dl.e0, s));
  Lc.go("init", k_ctl_init, 1, 1, s, ctl, (int32_t)cc, cc ? hi - lo : (owns_src ? 1u : 0u));
  fill<uint32_t>(Lc, nb.p, nw, 0u, s);
  fill<long long>(Lc, acc.p, kDP, 0ll, s);
  if (cc) {  // cc: label = id; round 0 is every owned row (dense), snapshot = id
    Lc.go("init", k_iota_from<L>, grid_n(nv), 256, s, lab.p, nv, (int64_t)0);
    Lc.go("init", k_iota_from<L>, grid_n(hi - lo), 256, s, snap.p, (int64_t)(hi - lo), (int64_t)lo);
    Lc.go("init", k_iota_from<L>, grid_n(hi - lo), 256, s, own.p, (int64_t)(hi - lo), (int64_t)lo);
  } else {
    fill<L>(Lc, lab.p, nv, inf, s);
    fill<L>(Lc, own.p, std::max<int64_t>(hi - lo, 1), inf, s);
    Lc.go("init", k_set1<L>, 1, 1, s, lab.p, p.source, (L)0);
    if (owns_src) {
      Lc.go("init", k_set1<uint32_t>, 1, 1, s, rb.q0.p, (int64_t)0, (uint32_t)p.source);
      Lc.go("init", k_set1<L>, 1, 1, s, snap.p, (int64_t)0, (L)0);
      Lc.go("init", k_set1<L>, 1, 1, s, own.p, p.source - lo, (L)0);
    }
  }
  std::vector<size_t> sc(D), sd(D), rc(D), rd(D);
  std::vector<unsigned long long> hc(kMaxParts + 1);
  std::vector<long long> mat((size_t)D * D);
  DBuf<long long> dmat((size_t)D * D);
  for (int64_t r = 0; r <= limit; ++r) {
    RoundCtx c{Lc, s, cudaGraphConditionalHandle{}, 0};
    bm_round(c, a, op, p.blocked != 0, classic, tsum.p, /*compact=*/false);
    Lc.go("dist", k_dp_collect, 1, 32, s, a, acc.p);
    // ---- mirrors -> masters: how much would travel?
    fill<unsigned long long>(Lc, cnt.p, kMaxParts + 1, 0ull, s);
    Lc.go("dist", k_dp_count, grid_n(nw), 256, s, (const uint32_t *)nb.p, nv, cuts, R, cnt.p);
    SG_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, sizeof(unsigned long long) * D, cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    std::fill(mat.begin(), mat.end(), 0);
    long long sent = 0;
    for (int q = 0; q < D; ++q) mat[(size_t)R * D + q] = (long long)hc[q], sent += (long long)hc[q];
    SG_CUDA(cudaMemcpyAsync(dmat.p, mat.data(), sizeof(long long) * D * D, cudaMemcpyHostToDevice, s));
    cm.allreduce(dmat.p, (size_t)D * D, CType::I64, COp::Sum, s);
    SG_CUDA(cudaMemcpyAsync(mat.data(), dmat.p, sizeof(long long) * D * D, cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    long long total = 0;
    for (long long x : mat) total += x;
    // the updates travel twice (to the owner, back to every mirror holder);
    // a dense all-reduce moves ~2 V labels per rank
    // (sg_params.reserved: 1 forces the sparse exchange, 2 the dense one)
    const bool sparse = D > 1 && (p.reserved == 1 ||
                                  (p.reserved != 2 && total * 2 * (4 + (long long)sizeof(L)) * D <
                                                          2 * nv * (long long)sizeof(L) * (D - 1)));
    if (D > 1 && sparse) {
      size_t off = 0;
      for (int q = 0; q < D; ++q) sd[q] = off, sc[q] = (size_t)mat[(size_t)R * D + q], off += sc[q];
      size_t roff = 0;
      for (int q = 0; q < D; ++q) rd[q] = roff, rc[q] = (size_t)mat[(size_t)q * D + R], roff += rc[q];
      std::vector<unsigned long long> cur(D);
      for (int q = 0; q < D; ++q) cur[q] = sd[q];
      SG_CUDA(cudaMemcpyAsync(cursor.p, cur.data(), sizeof(unsigned long long) * D,
                              cudaMemcpyHostToDevice, s));
      Lc.go("dist", k_dp_pack<L>, grid_n(nw), 256, s, (const uint32_t *)nb.p, (const L *)lab.p, nv,
            cuts, R, cursor.p, sids.p, svals.p);
      cm.group_begin();  // ids and labels in ONE grouped NCCL launch
      cm.alltoallv(sids.p, sc.data(), sd.data(), rids.p, rc.data(), rd.data(), CType::U32, s);
      cm.alltoallv(svals.p, sc.data(), sd.data(), rvals.p, rc.data(), rd.data(), LT, s);
      cm.group_end();
      if (roff)
        Lc.go("dist", k_dp_apply<L>, grid_n((int64_t)roff), 256, s, (const uint32_t *)rids.p,
              (const L *)rvals.p, (int64_t)roff, lab.p);
    } else if (D > 1) {
      cm.allreduce(lab.p, (size_t)nv, LT, COp::Min, s);
    }
    // ---- masters: changed rows -> next frontier (+ the mirrors' update list)
    Lc.go("dist", k_dp_diff<L>, grid_n(hi - lo), 256, s, (const L *)lab.p, own.p, lo, hi, rb.q0.p,
          snap.p, ctl, (const uint32_t *)(D > 1 ? mc.p : nullptr), uids.p, uvals.p, acc.p);
    if (D > 1 && sparse) {  // masters -> mirrors: every rank's changed rows to every rank
      uint32_t nch = 0;
      SG_CUDA(cudaMemcpyAsync(&nch, &ctl->nsize, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      SG_CUDA(cudaStreamSynchronize(s));
      std::vector<long long> per(D, 0);
      per[R] = nch;
      DBuf<long long> dper(D);
      SG_CUDA(cudaMemcpyAsync(dper.p, per.data(), sizeof(long long) * D, cudaMemcpyHostToDevice, s));
      cm.allreduce(dper.p, (size_t)D, CType::I64, COp::Sum, s);
      SG_CUDA(cudaMemcpyAsync(per.data(), dper.p, sizeof(long long) * D, cudaMemcpyDeviceToHost, s));
      SG_CUDA(cudaStreamSynchronize(s));
      size_t roff = 0;
      for (int q = 0; q < D; ++q) {
        sc[q] = q == R ? 0 : nch, sd[q] = 0;
        rc[q] = q == R ? 0 : (size_t)per[q], rd[q] = roff, roff += rc[q];
      }
      cm.group_begin();
      cm.alltoallv(uids.p, sc.data(), sd.data(), rids.p, rc.data(), rd.data(), CType::U32, s);
      cm.alltoallv(uvals.p, sc.data(), sd.data(), rvals.p, rc.data(), rd.data(), LT, s);
      cm.group_end();
      if (roff)
        Lc.go("dist", k_dp_apply<L>, grid_n((int64_t)roff), 256, s, (const uint32_t *)rids.p,
              (const L *)rvals.p, (int64_t)roff, lab.p);
    }
    fill<uint32_t>(Lc, nb.p, nw, 0u, s);
    SG_CUDA(cudaMemcpyAsync(cnt.p + kMaxParts, &sent, sizeof(long long), cudaMemcpyHostToDevice, s));
    Lc.go("dist", k_dp_next, 1, 32, s, (const Ctl *)ctl, acc.p, cnt.p + kMaxParts);
    cm.allreduce(acc.p, kDP, CType::I64, COp::Sum, s);
    Lc.go("advance", k_dp_advance, 1, 32, s, a, acc.p, lp);
    if (dl.done(ctl)) break;
  }
  DBuf<double> out(std::max<int64_t>(nv, 1));
  if (sizeof(L) == 4)
    Lc.go("labels", k_labels_u32, grid_n(nv), 256, s, (const uint32_t *)lab.p, nv, out.p);
  else
    Lc.go("labels", k_labels_f64bits, grid_n(nv), 256, s, (const unsigned long long *)lab.p, nv,
          out.p);
  SG_CUDA(cudaEventRecord(dl.e1, s));
  SG_CUDA(cudaEventSynchronize(dl.e1));
  float ms = 0;
  SG_CUDA(cudaEventElapsedTime(&ms, dl.e0, dl.e1));
  if (ms_out) *ms_out = ms;
  dist_results(rb, s, out.p, nv, rounds_out, cap, nrounds, labels_out, max_rounds);
}

}  // namespace

void run_push_dist(Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds, Comm &cm,
                   double *labels_out, sg_round *rounds_out, int64_t cap, int64_t *nrounds,
                   double *ms_out) {
  if (p.app == SG_APP_CC)
    return run_dist_push<0>(g, p, thr, max_rounds, cm, labels_out, rounds_out, cap, nrounds, ms_out);
  const bool weighted = p.app == SG_APP_SSSP && g.weighted;
  if (!weighted)  // bfs == unit-weight relaxation (same labels and rounds)
    return run_dist_push<1>(g, p, thr, max_rounds, cm, labels_out, rounds_out, cap, nrounds, ms_out);
  const double bound = (double)g.wmax * (double)std::max<int64_t>(g.nv - 1, 1);
  if (g.w32.p && bound < 4294967295.0)
    return run_dist_push<2>(g, p, thr, max_rounds, cm, labels_out, rounds_out, cap, nrounds, ms_out);
  return run_dist_push<3>(g, p, thr, max_rounds, cm, labels_out, rounds_out, cap, nrounds, ms_out);
}

}  // namespace sg
