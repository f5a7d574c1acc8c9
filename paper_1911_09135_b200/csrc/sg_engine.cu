// sg_engine.cu — the BSP driver (reference engine.py:190-246) on the device.
//
// One round = a fixed sequence of kernels whose sizes live in device memory
// (Ctl), captured once into a CUDA graph and replayed; the host only checks
// the `done` flag after batches of rounds (1, 2, 4, ... 32), and rounds
// issued past the end exit immediately.  Results: float64 labels + one
// RoundStat per round (frontier size, active edges, ... == RoundRecord).
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <unordered_map>

#include "sg_graph.cuh"
#include "sg_pull.cuh"

namespace sg {

std::atomic<int64_t> g_launches{0};
static thread_local std::string t_last_error;
void set_last_error(const std::string &m) { t_last_error = m; }

const SmInfo &sm_info() {
  static SmInfo info = [] {
    SmInfo s;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      s.device = dev;
      int n = 0;
      if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n)
        s.sms = n;
    }
    return s;
  }();
  return info;
}

namespace {

template <class K>
int occupancy_grid(K kernel, int block, int cap_per_sm = 8) {
  static std::mutex mu;
  static std::unordered_map<const void *, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find((const void *)kernel);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0));
  per_sm = std::max(1, std::min(per_sm, cap_per_sm));
  int g = persistent_grid(per_sm);
  cache[(const void *)kernel] = g;
  return g;
}

inline int grid_n(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_info().sms * 32));
}

// ------------------------------------------------------------ init kernels --
template <class T>
__global__ void k_fill(T *p, int64_t n, T v) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) p[i] = v;
}
__global__ void k_iota32(uint32_t *p, int64_t n) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    p[i] = (uint32_t)i;
}
template <class T>
__global__ void k_set1(T *p, int64_t i, T v) { p[i] = v; }

__global__ void k_labels_u32(const uint32_t *lab, int64_t n, double *out) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = lab[i] == kInf32 ? INFINITY : (double)lab[i];
}
__global__ void k_labels_alive(const uint8_t *a, int64_t n, double *out) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = a[i] ? 1.0 : 0.0;
}

// inv_outdeg (apps.py:158-161)
__global__ void k_inv_outdeg(const int64_t *off, int64_t n, double *inv) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += st) {
    int64_t d = off[v + 1] - off[v];
    inv[v] = d > 0 ? 1.0 / (double)d : 0.0;
  }
}
__global__ void k_pr_init(const double *inv, int64_t n, double omd, double *rank, double *aux) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += st) {
    rank[v] = omd;
    aux[v] = __dmul_rn(omd, inv[v]);  // round_aux of round 0 (apps.py:176-177)
  }
}
// gain[v] = sum_{u->v} inv[u] accumulated in CSC (== CSR edge) order, exactly
// as np.bincount does (apps.py:166-168): one warp per row loads 32 terms and
// every lane folds them sequentially through shuffles.
__global__ void k_pr_gain_max(const int64_t *off, const uint32_t *col, int64_t n,
                              const double *inv, unsigned long long *maxbits) {
  int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double best = 0.0;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    double acc = 0.0;
    for (int64_t b = off[v]; b < off[v + 1]; b += 32) {
      int64_t j = b + lane_id();
      double x = j < off[v + 1] ? inv[col[j]] : 0.0;
      int cnt = (int)min((int64_t)32, off[v + 1] - b);
      for (int t = 0; t < cnt; ++t) acc = __dadd_rn(acc, __shfl_sync(kFull, x, t));
    }
    best = acc > best ? acc : best;
  }
  if (lane_id() == 0 && best > 0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(best));
}

// static bins of a dense pull view (pr): CTA-bin rows and huge rows
__global__ void k_static_bins(const int64_t *off, uint32_t n, int64_t thr, uint32_t *largeq,
                              uint32_t *hugeq, Ctl *ctl) {
  uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < n; b += st) {
    uint64_t v = b + threadIdx.x;
    int64_t d = v < n ? off[v + 1] - off[v] : 0;
    bool huge = v < n && d >= thr;
    bool large = v < n && !huge && d >= (int64_t)kLarge;
    warp_append(huge, (uint32_t)v, hugeq, &ctl->nhuge);
    warp_append(large, (uint32_t)v, largeq, &ctl->nlarge);
  }
}

// ------------------------------------------------------- advance kernels --
// commit (snapshot := label for changed vertices) + round bookkeeping
template <class L, bool COMMIT>
__global__ void __launch_bounds__(256) k_push_advance(PushArgs a, L *lab, L *snap,
                                                      int64_t max_rounds) {
  __shared__ bool last;
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  const uint32_t nn = ctl->nsize;
  if (COMMIT) {
    const uint32_t *nq = a.q[(round + 1) & 1];
    int64_t st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += st) {
      uint32_t v = nq[i];
      snap[v] = lab[v];
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ctl->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x) return;
  RoundStat &s = a.stats[round];
  s.frontier_size = ctl->dense ? a.nv : ctl->fsize;
  s.active_edges = (long long)ctl->edges;
  s.huge_count = ctl->nhuge;
  s.huge_edges = (long long)ctl->huge_edges;
  s.large_count = ctl->nlarge;
  s.updated = nn;
  s.comm_sent = (long long)ctl->comm_sent;
  s.comm_broadcast = (long long)ctl->comm_bcast;
  ctl->fsize = nn;
  ctl->nsize = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = 0;
  ctl->edges = ctl->huge_edges = ctl->comm_sent = ctl->comm_bcast = 0;
  ctl->dense = 0;
  ctl->ticket = 0;
  ctl->round = round + 1;
  if (nn == 0) ctl->done = 1;
  else if ((int64_t)round + 1 >= max_rounds) ctl->error = SG_ECONVERGE, ctl->done = 1;
  __threadfence();
}

// kcore: record the count-phase stats, then kill the dying (apps.py:225)
__global__ void k_kcore_kill(PullArgs a, uint8_t *alive) {
  Ctl *ctl = a.ctl;
  if (ctl->done) return;
  const uint32_t nd = ctl->ndying;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += st)
    alive[a.dying[i]] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    RoundStat &s = a.stats[ctl->round];
    s.frontier_size = ctl->dense ? a.nv : ctl->fsize;
    s.active_edges = (long long)ctl->edges;
    s.huge_count = ctl->nhuge;
    s.huge_edges = (long long)ctl->huge_edges;
    s.large_count = ctl->nlarge;
    s.updated = nd;
    s.comm_sent = 0;
    s.comm_broadcast = 0;
    // the neighbour walk reuses the CTA-bin queue
    ctl->nlarge = ctl->nhuge = ctl->large_head = 0;
    ctl->huge_edges = 0;
  }
}

__global__ void k_kcore_advance(Ctl *ctl, int64_t max_rounds) {
  if (ctl->done) return;
  const uint32_t round = ctl->round;
  const uint32_t nd = ctl->ndying, nn = ctl->nsize;
  ctl->fsize = nn;
  ctl->nsize = 0;
  ctl->ndying = 0;
  ctl->nlarge = ctl->nhuge = ctl->large_head = 0;
  ctl->edges = ctl->huge_edges = 0;
  ctl->dense = 0;
  ctl->round = round + 1;
  if (nd == 0 || nn == 0) ctl->done = 1;  // apps.py:223-232
  else if ((int64_t)round + 1 >= max_rounds) ctl->error = SG_ECONVERGE, ctl->done = 1;
}

// ------------------------------------------------------------ run state --
struct RunBufs {
  DBuf<Ctl> ctl;
  DBuf<RoundStat> stats;
  int64_t stats_cap = 0;
  DBuf<uint32_t> q0, q1, largeq, hugeq, dying;
  DBuf<int64_t> hpre, hstart;
  DBuf<unsigned long long> hval;

  void alloc_common(int64_t nv, int64_t rounds_cap) {
    size_t n = (size_t)std::max<int64_t>(nv, 1);
    ctl.alloc(1);
    SG_CUDA(cudaMemset(ctl.p, 0, sizeof(Ctl)));
    stats_cap = rounds_cap;
    stats.alloc(rounds_cap);
    q0.alloc(n), q1.alloc(n), largeq.alloc(n), hugeq.alloc(n);
    hpre.alloc(n), hstart.alloc(n), hval.alloc(n);
  }
  PushArgs push_args(const View &v, int64_t thr) {
    PushArgs a{};
    a.off = v.off.p;
    a.col = v.col.p;
    a.nv = (uint32_t)v.nv;
    a.ctl = ctl.p;
    a.q[0] = q0.p, a.q[1] = q1.p;
    a.largeq = largeq.p, a.hugeq = hugeq.p;
    a.hpre = hpre.p, a.hstart = hstart.p, a.hval = hval.p;
    a.dying = dying.p;
    a.threshold = thr;
    a.src_mode = 0;
    a.stats = stats.p;
    return a;
  }
  PullArgs pull_args(const View &v, int64_t thr, int dyn) {
    PullArgs a{};
    a.off = v.off.p;
    a.col = v.col.p;
    a.nv = (uint32_t)v.nv;
    a.ctl = ctl.p;
    a.q[0] = q0.p, a.q[1] = q1.p;
    a.largeq = largeq.p, a.hugeq = hugeq.p;
    a.hpre = hpre.p, a.hstart = hstart.p;
    a.threshold = thr;
    a.dynamic_bins = dyn;
    a.dying = dying.p;
    a.stats = stats.p;
    return a;
  }
};

template <class T>
void fill(T *p, int64_t n, T v, cudaStream_t s) {
  if (n > 0) SG_LAUNCH(k_fill<T>, grid_n(n), 256, 0, s, p, n, v);
}

// Capture `round` once, replay until the device says done.
template <class F>
void bsp_loop(RunBufs &rb, F &&round, cudaStream_t s, int64_t max_rounds, int64_t *issued_out) {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  SG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  round(s);
  SG_CUDA(cudaStreamEndCapture(s, &graph));
  SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  Ctl *h = nullptr;
  SG_CUDA(cudaMallocHost(&h, sizeof(Ctl)));
  int64_t issued = 0, batch = 1;
  int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  bool ok = true;
  for (;;) {
    int64_t nb = std::min<int64_t>(batch, std::max<int64_t>(limit - issued, 1));
    for (int64_t b = 0; b < nb; ++b) {
      if (cudaGraphLaunch(exec, s) != cudaSuccess) { ok = false; break; }
      g_launches.fetch_add(4, std::memory_order_relaxed);
      ++issued;
    }
    if (!ok) break;
    if (cudaMemcpyAsync(h, rb.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) { ok = false; break; }
    if (h->done) break;
    if (issued >= limit) { ok = false; break; }
    batch = std::min<int64_t>(batch * 2, 32);
  }
  bool capped = !ok && issued >= limit;
  cudaFreeHost(h);
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  SG_CUDA(cudaGetLastError());
  if (capped) throw Error(SG_ECONVERGE, "round budget exhausted");
  if (!ok) SG_CUDA(cudaDeviceSynchronize());
  *issued_out = issued;
}

// ----------------------------------------------------------------- apps --
template <class Op>
void push_round(const PushArgs &a, const Op &op, bool blocked, cudaStream_t s) {
  SG_LAUNCH(k_push_twc<Op>, occupancy_grid(k_push_twc<Op>, kTB), kTB, 0, s, a, op);
  SG_LAUNCH(k_push_large<Op>, occupancy_grid(k_push_large<Op>, kTB), kTB, 0, s, a, op);
  if (a.threshold != std::numeric_limits<int64_t>::max()) {
    SG_LAUNCH(k_huge_prefix<Op>, 1, 1024, 0, s, a, op);
    if (blocked)
      SG_LAUNCH((k_push_lb<Op, true>), occupancy_grid(k_push_lb<Op, true>, kTB), kTB, 0, s, a, op);
    else
      SG_LAUNCH((k_push_lb<Op, false>), occupancy_grid(k_push_lb<Op, false>, kTB), kTB, 0, s, a,
                op);
  }
}

template <class Op>
void pull_round(const PullArgs &a, const Op &op, bool blocked, typename Op::A *hacc,
                cudaStream_t s) {
  SG_LAUNCH(k_pull_twc<Op>, occupancy_grid(k_pull_twc<Op>, kTB), kTB, 0, s, a, op);
  SG_LAUNCH(k_pull_large<Op>, occupancy_grid(k_pull_large<Op>, kTB), kTB, 0, s, a, op);
  if (a.threshold != std::numeric_limits<int64_t>::max()) {
    if (a.dynamic_bins) SG_LAUNCH(k_pull_prefix, 1, 1024, 0, s, a);
    if (blocked)
      SG_LAUNCH((k_pull_lb<Op, true>), occupancy_grid(k_pull_lb<Op, true>, kTB), kTB, 0, s, a, op,
                hacc);
    else
      SG_LAUNCH((k_pull_lb<Op, false>), occupancy_grid(k_pull_lb<Op, false>, kTB), kTB, 0, s, a,
                op, hacc);
  }
}

struct RunOut {
  DBuf<double> labels;
  int64_t rounds = 0;
};

void run_push_min(Graph &g, const sg_params &p, RunBufs &rb, RunOut &ro, cudaStream_t s,
                  int64_t thr, int64_t max_rounds) {
  const bool cc = p.app == SG_APP_CC;
  const View &v = cc ? g.sym() : g.csr;
  const int64_t nv = v.nv;
  rb.alloc_common(nv, std::min<int64_t>(max_rounds, 1 << 20));
  PushArgs a = rb.push_args(v, thr);
  Ctl init{};
  if (cc) {
    init.dense = 1;
    init.fsize = (uint32_t)nv;
  } else {
    init.fsize = 1;
    SG_LAUNCH(k_set1<uint32_t>, 1, 1, 0, s, rb.q0.p, 0, (uint32_t)p.source);
  }
  SG_CUDA(cudaMemcpyAsync(rb.ctl.p, &init, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  ro.labels.alloc(std::max<int64_t>(nv, 1));
  const bool blocked = p.blocked != 0;

  if (p.app == SG_APP_BFS) {
    DBuf<uint32_t> lab(std::max<int64_t>(nv, 1)), vis((nv + 31) / 32 + 1);
    fill<uint32_t>(lab.p, nv, kInf32, s);
    fill<uint32_t>(vis.p, (nv + 31) / 32 + 1, 0u, s);
    SG_LAUNCH(k_set1<uint32_t>, 1, 1, 0, s, lab.p, p.source, 0u);
    SG_LAUNCH(k_set1<uint32_t>, 1, 1, 0, s, vis.p, p.source >> 5, 1u << (p.source & 31));
    OpBfs op{lab.p, vis.p};
    bsp_loop(rb, [&](cudaStream_t st) {
      push_round(a, op, blocked, st);
      SG_LAUNCH((k_push_advance<uint32_t, false>), 1, 256, 0, st, a, lab.p, lab.p, max_rounds);
    }, s, max_rounds, &ro.rounds);
    SG_LAUNCH(k_labels_u32, grid_n(nv), 256, 0, s, lab.p, nv, ro.labels.p);
    SG_CUDA(cudaStreamSynchronize(s));
    return;
  }

  // sssp / cc: 32-bit labels when every path sum provably fits, else f64 bits
  bool weighted = p.app == SG_APP_SSSP && g.weighted;
  bool use32 = true;
  if (weighted) {
    if (g.wmin < 0) throw Error(SG_ECONFIG, "sssp requires non-negative weights");
    double bound = (double)g.wmax * (double)std::max<int64_t>(nv - 1, 1);
    use32 = g.w32.p != nullptr && bound < 4294967295.0;
  }
  if (use32) {
    DBuf<uint32_t> lab(std::max<int64_t>(nv, 1)), snap(std::max<int64_t>(nv, 1));
    if (cc) {
      SG_LAUNCH(k_iota32, grid_n(nv), 256, 0, s, lab.p, nv);
      SG_LAUNCH(k_iota32, grid_n(nv), 256, 0, s, snap.p, nv);
    } else {
      fill<uint32_t>(lab.p, nv, kInf32, s);
      fill<uint32_t>(snap.p, nv, kInf32, s);
      SG_LAUNCH(k_set1<uint32_t>, 1, 1, 0, s, lab.p, p.source, 0u);
      SG_LAUNCH(k_set1<uint32_t>, 1, 1, 0, s, snap.p, p.source, 0u);
    }
    auto go = [&](auto op) {
      using Op = decltype(op);
      bsp_loop(rb, [&](cudaStream_t st) {
        push_round(a, op, blocked, st);
        SG_LAUNCH((k_push_advance<uint32_t, true>), grid_n(nv, 256), 256, 0, st, a, lab.p,
                  snap.p, max_rounds);
      }, s, max_rounds, &ro.rounds);
      (void)sizeof(Op);
    };
    if (cc) go(OpMin32<0>{lab.p, snap.p, nullptr});
    else if (!weighted) go(OpMin32<1>{lab.p, snap.p, nullptr});
    else go(OpMin32<2>{lab.p, snap.p, g.w32.p});
    SG_LAUNCH(k_labels_u32, grid_n(nv), 256, 0, s, lab.p, nv, ro.labels.p);
  } else {
    DBuf<unsigned long long> lab(std::max<int64_t>(nv, 1)), snap(std::max<int64_t>(nv, 1));
    const unsigned long long inf = 0x7ff0000000000000ull;
    fill<unsigned long long>(lab.p, nv, inf, s);
    fill<unsigned long long>(snap.p, nv, inf, s);
    SG_LAUNCH(k_set1<unsigned long long>, 1, 1, 0, s, lab.p, p.source, 0ull);
    SG_LAUNCH(k_set1<unsigned long long>, 1, 1, 0, s, snap.p, p.source, 0ull);
    OpMinF64 op{lab.p, snap.p, weighted ? g.w64.p : nullptr};
    bsp_loop(rb, [&](cudaStream_t st) {
      push_round(a, op, blocked, st);
      SG_LAUNCH((k_push_advance<unsigned long long, true>), grid_n(nv, 256), 256, 0, st, a,
                lab.p, snap.p, max_rounds);
    }, s, max_rounds, &ro.rounds);
    SG_CUDA(cudaMemcpyAsync(ro.labels.p, lab.p, sizeof(double) * nv, cudaMemcpyDeviceToDevice, s));
  }
  SG_CUDA(cudaStreamSynchronize(s));
}

void run_pr(Graph &g, const sg_params &p, RunBufs &rb, RunOut &ro, cudaStream_t s, int64_t thr,
            int64_t max_rounds) {
  const View &v = g.csc();
  const int64_t nv = v.nv;
  rb.alloc_common(nv, std::min<int64_t>(max_rounds, 1 << 20));
  PullArgs a = rb.pull_args(v, thr, 0);
  ro.labels.alloc(std::max<int64_t>(nv, 1));
  DBuf<double> inv(std::max<int64_t>(nv, 1)), aux0(std::max<int64_t>(nv, 1)),
      aux1(std::max<int64_t>(nv, 1)), hacc(std::max<int64_t>(nv, 1));
  DBuf<unsigned long long> gmax(1);
  const double d = p.damping, omd = 1.0 - p.damping;
  SG_LAUNCH(k_inv_outdeg, grid_n(nv), 256, 0, s, g.csr.off.p, nv, inv.p);
  SG_LAUNCH(k_pr_init, grid_n(nv), 256, 0, s, inv.p, nv, omd, ro.labels.p, aux0.p);
  fill<double>(hacc.p, nv, 0.0, s);
  SG_CUDA(cudaMemsetAsync(gmax.p, 0, sizeof(unsigned long long), s));
  double worst = 0.0;
  if (g.ne) {
    SG_LAUNCH(k_pr_gain_max, grid_n(nv * 32), 256, 0, s, v.off.p, v.col.p, nv, inv.p, gmax.p);
    unsigned long long gb = 0;
    SG_CUDA(cudaMemcpyAsync(&gb, gmax.p, sizeof(gb), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    double gm;
    std::memcpy(&gm, &gb, 8);
    worst = d * gm;
  }
  const double eps_stop = p.tol / std::max(1.0, worst);  // apps.py:171
  Ctl init{};
  init.dense = 1;
  init.fsize = (uint32_t)nv;
  SG_CUDA(cudaMemcpyAsync(rb.ctl.p, &init, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  SG_LAUNCH(k_static_bins, grid_n(nv), 256, 0, s, v.off.p, (uint32_t)nv, thr, rb.largeq.p,
            rb.hugeq.p, rb.ctl.p);
  if (thr != std::numeric_limits<int64_t>::max()) SG_LAUNCH(k_pull_prefix, 1, 1024, 0, s, a);
  PrOp op{aux0.p, aux1.p, aux1.p, aux0.p, ro.labels.p, inv.p, d, omd};
  const bool blocked = p.blocked != 0;
  bsp_loop(rb, [&](cudaStream_t st) {
    pull_round(a, op, blocked, hacc.p, st);
    SG_LAUNCH((k_pull_finish<PrOp, true>), 1, 1024, 0, st, a, op, hacc.p, eps_stop, v.ne,
              max_rounds);
  }, s, max_rounds, &ro.rounds);
  SG_CUDA(cudaStreamSynchronize(s));
}

void run_kcore(Graph &g, const sg_params &p, RunBufs &rb, RunOut &ro, cudaStream_t s, int64_t thr,
               int64_t max_rounds) {
  if (p.k < 1) throw Error(SG_ECONFIG, "k must be >= 1");
  const View &v = g.sym();  // count rows: CSC(sym) and CSR(sym) rows hold the same multiset
  const int64_t nv = v.nv;
  rb.alloc_common(nv, std::min<int64_t>(max_rounds, 1 << 20));
  rb.dying.alloc(std::max<int64_t>(nv, 1));
  PullArgs a = rb.pull_args(v, thr, 1);
  PushArgs w = rb.push_args(v, std::numeric_limits<int64_t>::max());
  w.src_mode = 1;
  ro.labels.alloc(std::max<int64_t>(nv, 1));
  DBuf<uint8_t> alive(std::max<int64_t>(nv, 1));
  DBuf<uint32_t> mark(std::max<int64_t>(nv, 1)), hcnt(std::max<int64_t>(nv, 1));
  fill<uint8_t>(alive.p, nv, (uint8_t)1, s);
  fill<uint32_t>(mark.p, nv, 0u, s);
  fill<uint32_t>(hcnt.p, nv, 0u, s);
  Ctl init{};
  init.dense = 1;
  init.fsize = (uint32_t)nv;
  SG_CUDA(cudaMemcpyAsync(rb.ctl.p, &init, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  KcOp op{alive.p, (uint32_t)std::min<int64_t>(p.k, 0xffffffffLL)};
  OpMark mop{alive.p, mark.p};
  const bool blocked = p.blocked != 0;
  bsp_loop(rb, [&](cudaStream_t st) {
    pull_round(a, op, blocked, hcnt.p, st);
    if (thr != std::numeric_limits<int64_t>::max())
      SG_LAUNCH((k_pull_finish<KcOp, false>), 1, 1024, 0, st, a, op, hcnt.p, 0.0, v.ne,
                max_rounds);
    SG_LAUNCH(k_kcore_kill, grid_n(nv), 256, 0, st, a, alive.p);
    SG_LAUNCH(k_push_twc<OpMark>, occupancy_grid(k_push_twc<OpMark>, kTB), kTB, 0, st, w, mop);
    SG_LAUNCH(k_push_large<OpMark>, occupancy_grid(k_push_large<OpMark>, kTB), kTB, 0, st, w,
              mop);
    SG_LAUNCH(k_kcore_advance, 1, 1, 0, st, rb.ctl.p, max_rounds);
  }, s, max_rounds, &ro.rounds);
  SG_LAUNCH(k_labels_alive, grid_n(nv), 256, 0, s, alive.p, nv, ro.labels.p);
  SG_CUDA(cudaStreamSynchronize(s));
}

void run_app(Graph &g, const sg_params &p, double *labels_out, sg_round *rounds_out, int64_t cap,
             int64_t *nrounds, double *ms_out) {
  if (p.app < SG_APP_BFS || p.app > SG_APP_KCORE) throw Error(SG_ECONFIG, "unknown app");
  if (p.devices < 1) throw Error(SG_ECONFIG, "device count must be >= 1");
  if (g.nv > 0x7fffffffLL) throw Error(SG_ERANGE, "vertex ids must fit int32");
  if ((p.app == SG_APP_BFS || p.app == SG_APP_SSSP) && (p.source < 0 || p.source >= g.nv))
    throw Error(SG_ECONFIG, "source " + std::to_string(p.source) + " outside graph");
  if (p.app == SG_APP_PR && !(p.damping > 0.0 && p.damping < 1.0))
    throw Error(SG_ECONFIG, "damping must be in (0, 1)");
  if (p.app == SG_APP_PR && !(p.tol > 0.0)) throw Error(SG_ECONFIG, "tolerance must be positive");
  if (p.app == SG_APP_SSSP && g.weighted && g.wmin < 0)
    throw Error(SG_ECONFIG, "sssp requires non-negative weights");
  int64_t max_rounds = p.max_rounds > 0 ? p.max_rounds : 10 * std::max<int64_t>(g.nv, 1) + 256;
  int64_t thr = p.sched == SG_SCHED_TWC ? std::numeric_limits<int64_t>::max()
                                        : std::max<int64_t>(1, p.threshold);
  // lazily built views (cached on the graph, like graph.py:102/117) are not timed
  if (p.app == SG_APP_CC || p.app == SG_APP_KCORE) g.sym();
  if (p.app == SG_APP_PR) g.csc();
  *nrounds = 0;
  if (g.nv == 0) {
    if (ms_out) *ms_out = 0.0;
    return;
  }
  cudaStream_t s;
  SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  SG_CUDA(cudaEventCreate(&e0));
  SG_CUDA(cudaEventCreate(&e1));
  RunBufs rb;
  RunOut ro;
  try {
    SG_CUDA(cudaEventRecord(e0, s));
    switch (p.app) {
      case SG_APP_BFS:
      case SG_APP_SSSP:
      case SG_APP_CC: run_push_min(g, p, rb, ro, s, thr, max_rounds); break;
      case SG_APP_PR: run_pr(g, p, rb, ro, s, thr, max_rounds); break;
      case SG_APP_KCORE: run_kcore(g, p, rb, ro, s, thr, max_rounds); break;
    }
    SG_CUDA(cudaEventRecord(e1, s));
    SG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms_out) *ms_out = ms;
    Ctl h;
    SG_CUDA(cudaMemcpy(&h, rb.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
    int64_t rounds = h.round;
    std::vector<RoundStat> st((size_t)std::min<int64_t>(rounds, rb.stats_cap));
    if (!st.empty())
      SG_CUDA(cudaMemcpy(st.data(), rb.stats.p, sizeof(RoundStat) * st.size(),
                         cudaMemcpyDeviceToHost));
    if (rounds_out)
      std::memcpy(rounds_out, st.data(), sizeof(RoundStat) * (size_t)std::min<int64_t>(cap, (int64_t)st.size()));
    *nrounds = rounds;
    if (labels_out)
      SG_CUDA(cudaMemcpy(labels_out, ro.labels.p, sizeof(double) * g.nv, cudaMemcpyDeviceToHost));
    if (h.error) throw Error(h.error, "did not converge within " + std::to_string(max_rounds) +
                                          " rounds");
  } catch (...) {
    cudaStreamSynchronize(s);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
}

}  // namespace
}  // namespace sg

// ====================================================================== C ABI
using sg::Error;

extern "C" {

const char *sg_last_error(void) { return sg::t_last_error.c_str(); }

int64_t sg_kernel_launches(void) { return sg::g_launches.load(); }

int sg_device_count(int *count) {
  return sg::guard([&] { SG_CUDA(cudaGetDeviceCount(count)); });
}

int sg_graph_create(const int64_t *offsets, const int32_t *targets, const int64_t *weights,
                    int64_t nv, int64_t ne, sg_graph **out) {
  return sg::guard([&] {
    if (nv < 0 || ne < 0) throw Error(SG_ECONFIG, "negative size");
    if (nv > 0x7fffffffLL) throw Error(SG_ERANGE, "vertex ids must fit int32");
    if (offsets[0] != 0 || offsets[nv] != ne)
      throw Error(SG_ECONFIG, "offsets must have num_vertices+1 entries starting at 0 and end at num_edges");
    auto g = std::make_shared<sg::Graph>();
    g->nv = nv, g->ne = ne;
    g->csr.nv = nv, g->csr.ne = ne;
    g->csr.off.alloc(nv + 1);
    g->csr.col.alloc(ne ? ne : 1);
    SG_CUDA(cudaMemcpy(g->csr.off.p, offsets, sizeof(int64_t) * (nv + 1), cudaMemcpyHostToDevice));
    if (ne)
      SG_CUDA(cudaMemcpy(g->csr.col.p, targets, sizeof(int32_t) * ne, cudaMemcpyHostToDevice));
    if (weights) {
      g->w64.alloc(ne ? ne : 1);
      if (ne)
        SG_CUDA(cudaMemcpy(g->w64.p, weights, sizeof(int64_t) * ne, cudaMemcpyHostToDevice));
      sg::weights_finalize(*g);
    }
    *out = new sg_graph{g};
  });
}

int sg_graph_create_rmat(int32_t scale, int64_t edge_factor, const uint64_t pcg[4],
                         const double cuts[3], sg_graph **out) {
  return sg::guard([&] {
    if (scale < 1 || scale > 31) throw Error(SG_ECONFIG, "scale must be in [1, 31]");
    if (edge_factor < 0) throw Error(SG_ECONFIG, "edge_factor must be >= 0");
    int64_t nv = (int64_t)1 << scale, ne = edge_factor * nv;
    auto g = std::make_shared<sg::Graph>();
    g->nv = nv, g->ne = ne;
    sg::DBuf<uint32_t> src(ne ? ne : 1), dst(ne ? ne : 1);
    if (ne) sg::rmat_pairs_device(scale, ne, pcg, cuts, src.p, dst.p);
    sg::build_csr_from_pairs(g->csr, nv, src.p, dst.p, ne, scale);
    *out = new sg_graph{g};
  });
}

int sg_graph_attach_random_weights(sg_graph *gh, const uint64_t pcg[4], int64_t low, int64_t high,
                                   sg_graph **out) {
  return sg::guard([&] {
    int64_t range = high - low + 1;
    int j = 0;
    while (j <= 32 && ((int64_t)1 << j) < range) ++j;
    if (range < 1 || j > 32 || ((int64_t)1 << j) != range)
      throw Error(SG_ECONFIG, "device weights need a power-of-two range <= 2^32");
    auto g = std::make_shared<sg::Graph>();
    const sg::Graph &src = *gh->g;
    g->nv = src.nv, g->ne = src.ne;
    g->csr.nv = src.nv, g->csr.ne = src.ne;
    g->csr.off.alloc(src.nv + 1);
    g->csr.col.alloc(src.ne ? src.ne : 1);
    SG_CUDA(cudaMemcpy(g->csr.off.p, src.csr.off.p, sizeof(int64_t) * (src.nv + 1),
                       cudaMemcpyDeviceToDevice));
    if (src.ne)
      SG_CUDA(cudaMemcpy(g->csr.col.p, src.csr.col.p, sizeof(uint32_t) * src.ne,
                         cudaMemcpyDeviceToDevice));
    g->w64.alloc(src.ne ? src.ne : 1);
    sg::random_weights_device(src.ne, pcg, low, j, g->w64.p);
    sg::weights_finalize(*g);
    *out = new sg_graph{g};
  });
}

int sg_graph_with_weights(sg_graph *gh, const int64_t *weights, sg_graph **out) {
  return sg::guard([&] {
    auto g = std::make_shared<sg::Graph>();
    const sg::Graph &src = *gh->g;
    g->nv = src.nv, g->ne = src.ne;
    g->csr.nv = src.nv, g->csr.ne = src.ne;
    g->csr.off.alloc(src.nv + 1);
    g->csr.col.alloc(src.ne ? src.ne : 1);
    SG_CUDA(cudaMemcpy(g->csr.off.p, src.csr.off.p, sizeof(int64_t) * (src.nv + 1),
                       cudaMemcpyDeviceToDevice));
    if (src.ne)
      SG_CUDA(cudaMemcpy(g->csr.col.p, src.csr.col.p, sizeof(uint32_t) * src.ne,
                         cudaMemcpyDeviceToDevice));
    g->w64.alloc(src.ne ? src.ne : 1);
    if (src.ne)
      SG_CUDA(cudaMemcpy(g->w64.p, weights, sizeof(int64_t) * src.ne, cudaMemcpyHostToDevice));
    sg::weights_finalize(*g);
    *out = new sg_graph{g};
  });
}

int sg_graph_info(sg_graph *g, int64_t *nv, int64_t *ne, int32_t *weighted) {
  return sg::guard([&] {
    if (nv) *nv = g->g->nv;
    if (ne) *ne = g->g->ne;
    if (weighted) *weighted = g->g->weighted;
  });
}

int sg_graph_view_size(sg_graph *g, int32_t which, int64_t *ne) {
  return sg::guard([&] {
    *ne = which == 2 ? 2 * g->g->ne : g->g->ne;
  });
}

int sg_graph_download(sg_graph *gh, int32_t which, int64_t *offsets, int32_t *targets,
                      int64_t *weights) {
  return sg::guard([&] {
    sg::Graph &g = *gh->g;
    const sg::View &v = which == 0 ? g.csr : which == 1 ? g.csc() : g.sym();
    if (offsets)
      SG_CUDA(cudaMemcpy(offsets, v.off.p, sizeof(int64_t) * (v.nv + 1), cudaMemcpyDeviceToHost));
    if (targets && v.ne)
      SG_CUDA(cudaMemcpy(targets, v.col.p, sizeof(int32_t) * v.ne, cudaMemcpyDeviceToHost));
    if (weights) {
      if (which != 0) throw Error(SG_ECONFIG, "weights are only downloadable for the CSR view");
      if (!g.weighted) throw Error(SG_ECONFIG, "graph is unweighted");
      if (g.ne)
        SG_CUDA(cudaMemcpy(weights, g.w64.p, sizeof(int64_t) * g.ne, cudaMemcpyDeviceToHost));
    }
  });
}

void sg_graph_destroy(sg_graph *g) { delete g; }

int sg_run(sg_graph *g, const sg_params *p, double *labels_out, sg_round *rounds_out,
           int64_t rounds_cap, int64_t *nrounds, double *ms_out) {
  return sg::guard([&] {
    sg::run_app(*g->g, *p, labels_out, rounds_out, rounds_cap, nrounds, ms_out);
  });
}

}  // extern "C"
