// sg_engine.cu — the BSP driver (reference engine.py:190-246) on the device.
//
// A round is a fixed sequence of kernels whose sizes live in device memory
// (Ctl).  It is captured once as the body of a CUDA-graph WHILE node; the
// round's last kernel evaluates the loop test (frontier empty / pr converged
// / round budget) and sets the node's condition, so the complete BSP loop is
// ONE graph launch with no host round trip.  SG_FLAG_PROFILE instead drives
// rounds from the host with CUDA events around every kernel (per-kernel
// times for the roofline report).  Results: float64 labels + one RoundStat
// per round (frontier size, active edges, ... == RoundRecord).

#include <cstdlib>
#include <thread>
#include <cub/device/device_scan.cuh>

#include "sg_runtime.cuh"
#include "sg_prx.cuh"


namespace sg {

std::atomic<int64_t> g_launches{0};
static thread_local std::string t_last_error;
void set_last_error(const std::string &m) { t_last_error = m; }

namespace {
struct DevPool {
  std::mutex mu;
  std::multimap<size_t, void *> free_blocks;
  std::unordered_map<void *, size_t> block_size;
};
DevPool &dev_pool() {
  static DevPool *p = new DevPool;  // intentionally leaked: usable during static destruction
  return *p;
}
size_t pool_round(size_t b) {
  const size_t g = b >= ((size_t)1 << 20) ? ((size_t)2 << 20) : 512;
  return (b + g - 1) / g * g;
}
}  // namespace

void *dev_alloc(size_t bytes) {
  DevPool &P = dev_pool();
  const size_t b = pool_round(bytes);
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.free_blocks.lower_bound(b);
    if (it != P.free_blocks.end() && it->first <= b + b / 8) {  // <= 12.5 % slack
      void *p = it->second;
      P.free_blocks.erase(it);
      return p;
    }
  }
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, b);
  if (e != cudaSuccess) {
    cudaGetLastError();
    dev_release_cached();
    e = cudaMalloc(&p, b);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(SG_ENOMEM, "cudaMalloc(" + std::to_string(b) + " B): " + cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lk(P.mu);
  P.block_size[p] = b;
  return p;
}

void dev_free(void *p) {
  DevPool &P = dev_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  auto it = P.block_size.find(p);
  if (it == P.block_size.end()) return;
  P.free_blocks.emplace(it->second, p);
}

// pinned host blocks for result buffers (cudaHostAlloc is slow: cache them)
namespace {
DevPool &host_pool() {
  static DevPool *p = new DevPool;
  return *p;
}
}  // namespace

void *host_alloc(size_t bytes) {
  DevPool &P = host_pool();
  size_t b = (size_t)1 << 16;  // power-of-two classes: pinning is slow, reuse matters
  while (b < bytes) b <<= 1;
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.free_blocks.find(b);
    if (it != P.free_blocks.end()) {
      void *p = it->second;
      P.free_blocks.erase(it);
      return p;
    }
  }
  void *p = nullptr;
  SG_CUDA(cudaHostAlloc(&p, b, cudaHostAllocDefault));
  std::lock_guard<std::mutex> lk(P.mu);
  P.block_size[p] = b;
  return p;
}

void host_free(void *p) {
  DevPool &P = host_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  auto it = P.block_size.find(p);
  if (it == P.block_size.end()) return;
  P.free_blocks.emplace(it->second, p);
}

void dev_release_cached() {
  DevPool &P = dev_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  cudaDeviceSynchronize();
  for (auto &kv : P.free_blocks) {
    cudaFree(kv.second);
    P.block_size.erase(kv.second);
  }
  P.free_blocks.clear();
}

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

}  // namespace sg

namespace sg {
namespace {

// old id of every vertex of a relabeled store (nullptr: identity); cc's initial
// labels are the vertex ids of the reference's numbering (apps.py:121-124)
// cc's streaming round 0 needs the row id of every symmetrized edge (4 B /
// edge, cached on the graph): built only when it fits with room to spare
// (a relabeled run also needs the original numbering's symmetrized rows; a
// graph relabeled before any cc run has not built them yet: build them too
// when they fit, ~3x their size with the sort's temporaries)
const uint32_t *maybe_sym_src(Graph &g) {
  if (g.sym_src_.p) return g.sym_src_.p;
  if (g.is_part()) return nullptr;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  const size_t ne2 = (size_t)std::max<int64_t>(2 * g.ne, 1);
  const size_t src_bytes = sizeof(uint32_t) * ne2;
  const size_t sym_bytes = g.sym_ ? 0 : 3 * (sizeof(uint32_t) * ne2 + 8 * (size_t)(g.nv + 1));
  if (fr < src_bytes + src_bytes / 2 + sym_bytes + ((size_t)2 << 30)) return nullptr;
  g.sym();
  return g.sym_src();
}

struct Layout {
  const uint32_t *perm = nullptr;  // new -> old
  const uint32_t *inv = nullptr;   // old -> new
  int64_t zout = -1, zsym = -1;    // first id without out-edges (CSR / symmetrized), -1: none known
  int64_t zin = -1;                // first id without in-edges (pull layouts), -1: none known
  const View *orig_sym = nullptr;  // relabeled cc: the original numbering's symmetrized rows
  const uint32_t *orig_src = nullptr;  // ... and their edges' row ids
};


__global__ void k_copy_u32(const uint32_t *__restrict__ a, int64_t n, uint32_t *__restrict__ b) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) b[i] = a[i];
}

// labels back to the reference's numbering: out[v] = lab[inv[v]]
__global__ void k_unpermute(const double *__restrict__ lab, const uint32_t *__restrict__ inv,
                            int64_t n, double *__restrict__ out) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = lab[inv[i]];
}

void prep_push_min(Program &P, Graph &g, const sg_params &p, RunBufs &rb, double *labels_d,
                   int64_t thr, int64_t max_rounds, const Layout &lay) {
  const bool classic = (p.flags & SG_FLAG_TWC_CLASSIC) != 0;
  const bool cc = p.app == SG_APP_CC;
  const View &v = cc ? g.sym() : g.csr;
  const int64_t nv = v.nv;
  rb.alloc_common(nv, stats_cap(max_rounds));
  PushArgs a = rb.push_args(v, thr);
  a.q[1] = a.q[0];  // one frontier array: k_bm_compact rewrites it after the round
  if (lay.perm && p.devices == 1) {  // relabeled store: edgeless vertices are numbered last
    const int64_t z = cc ? lay.zsym : lay.zout;
    if (z >= 0 && z <= nv) {
      a.zlo = (uint32_t)z;
      if (cc) a.dense_n = (uint32_t)z;  // round 0 (all of V) skips the isolated tail
    }
  }
  a.sched = p.sched == SG_SCHED_LB ? 1 : p.sched == SG_SCHED_VERTEX ? 2 : p.sched == SG_SCHED_EDGE ? 3 : 0;
  long long *tsum = a.sched == 1 || a.sched == 3 ? P.buf<long long>((nv + kFT - 1) / kFT + 1) : nullptr;
  const bool blocked = p.blocked != 0;
  const int64_t src = p.source;
  Ctl *ctl = rb.ctl.p;
  uint32_t *q0 = rb.q0.p;
  const int64_t nw = (nv + 31) / 32 + 1;
  auto init_ctl = [=](Launcher &L, cudaStream_t s) {
    L.go("init", k_ctl_init, 1, 1, s, ctl, (int32_t)cc, cc ? (uint32_t)nv : 1u);
    if (!cc) L.go("init", k_set1<uint32_t>, 1, 1, s, q0, (int64_t)0, (uint32_t)src);
  };
  auto set_round = [&](auto op) {
    P.round = [=, &rb](RoundCtx &c) {
      bm_round(c, a, op, blocked, classic, tsum);
      c.L.go_pdl("advance", k_push_advance, 1, 32, c.s, a, loop_of(rb, max_rounds, c));
    };
  };

  if (p.app == SG_APP_BFS) {
    uint32_t *lab = P.buf<uint32_t>(nv), *vis = P.buf<uint32_t>(nw), *prev = P.buf<uint32_t>(nw);
    P.init = [=](Launcher &L, cudaStream_t s) {
      init_ctl(L, s);
      fill<uint32_t>(L, lab, nv, kInf32, s);
      fill<uint32_t>(L, vis, nw, 0u, s);
      fill<uint32_t>(L, prev, nw, 0u, s);
      L.go("init", k_set1<uint32_t>, 1, 1, s, lab, src, 0u);
      L.go("init", k_set1<uint32_t>, 1, 1, s, vis, src >> 5, 1u << (src & 31));
      L.go("init", k_set1<uint32_t>, 1, 1, s, prev, src >> 5, 1u << (src & 31));
    };
    set_round(BmBfs{lab, vis, prev});
    P.unpermuted = P.inv != nullptr;
    P.finish = [=, inv = P.inv, out = P.out](Launcher &L, cudaStream_t s) {
      if (inv) L.go("labels", k_labels_u32_inv, grid_n(nv), 256, s, (const uint32_t *)lab, inv, nv, out);
      else L.go("labels", k_labels_u32, grid_n(nv), 256, s, lab, nv, labels_d);
    };
    return;
  }
  // sssp / cc: 32-bit labels when every path sum provably fits, else f64 bits
  const bool weighted = p.app == SG_APP_SSSP && g.weighted;
  bool use32 = true;
  if (weighted) {
    double bound = (double)g.wmax * (double)std::max<int64_t>(nv - 1, 1);
    use32 = g.w32.p != nullptr && bound < 4294967295.0;
  }
  uint32_t *nb = P.buf<uint32_t>(nw);
  const uint32_t *perm = lay.perm;
  if (use32) {
    uint32_t *lab = P.buf<uint32_t>(nv), *snap = P.buf<uint32_t>(nv);
    P.init = [=](Launcher &L, cudaStream_t s) {
      init_ctl(L, s);
      fill<uint32_t>(L, nb, nw, 0u, s);
      if (cc && perm) {
        L.go("init", k_copy_u32, grid_n(nv), 256, s, perm, nv, lab);
        L.go("init", k_copy_u32, grid_n(nv), 256, s, perm, nv, snap);
      } else if (cc) {
        L.go("init", k_iota, grid_n(nv), 256, s, lab, nv);
        L.go("init", k_iota, grid_n(nv), 256, s, snap, nv);  // dense round 0: snap[i] = i
      } else {
        fill<uint32_t>(L, lab, nv, kInf32, s);
        L.go("init", k_set1<uint32_t>, 1, 1, s, lab, src, 0u);
        L.go("init", k_set1<uint32_t>, 1, 1, s, snap, (int64_t)0, 0u);
      }
    };
    if (cc) set_round(BmMin<0>{lab, nullptr, nullptr, snap, nb});
    else if (!weighted) set_round(BmMin<1>{lab, nullptr, nullptr, snap, nb});
    else set_round(BmMin<2>{lab, g.w32.p, nullptr, snap, nb});
    // cc round 0 as one streaming pull over the original-numbering rows
    // (k_cc_dense, sg_bm.cuh) when those rows are at hand; SG_CC_DENSE=0: push
    static const bool cc_dense_env = [] {
      const char *e = std::getenv("SG_CC_DENSE");
      return e ? std::atoi(e) != 0 : true;
    }();
    const View *ov = !cc ? nullptr : lay.perm ? lay.orig_sym : &v;
    const uint32_t *src0 = !cc || !cc_dense_env || a.sched != 0 ? nullptr
                           : lay.perm ? lay.orig_src : maybe_sym_src(g);
    if (cc && ov && src0) {
      CcDenseArgs ca{ov->off.p, ov->col.p, src0, nv, ov->ne, lay.perm ? lay.inv : nullptr,
                     lab, nb, ctl, thr};
      const BmMin<0> op0{lab, nullptr, nullptr, snap, nb};
      auto base_init = P.init;
      const int64_t mr = max_rounds;
      P.init = [=, &rb](Launcher &L, cudaStream_t s) {
        base_init(L, s);
        L.go("cc_dense", k_cc_dense_bins, grid_n(nv), kTB, s, ca);
        L.go("cc_dense", k_cc_dense, occupancy_grid(k_cc_dense, kTB), kTB, s, ca);
        L.go("compact", k_bm_compact<BmMin<0>>, occupancy_grid(k_bm_compact<BmMin<0>>, kTB), kTB,
             s, a, op0);
        L.go("advance", k_push_advance_plain, 1, 32, s, a,
             Loop{std::min<int64_t>(mr, rb.stats_cap), mr, cudaGraphConditionalHandle{}, 0});
      };
    }
    P.unpermuted = P.inv != nullptr;
    P.finish = [=, inv = P.inv, out = P.out](Launcher &L, cudaStream_t s) {
      if (inv) L.go("labels", k_labels_u32_inv, grid_n(nv), 256, s, (const uint32_t *)lab, inv, nv, out);
      else L.go("labels", k_labels_u32, grid_n(nv), 256, s, lab, nv, labels_d);
    };
  } else {
    using U = unsigned long long;
    U *lab = P.buf<U>(nv), *snap = P.buf<U>(nv);
    const U inf = 0x7ff0000000000000ull;
    P.init = [=](Launcher &L, cudaStream_t s) {
      init_ctl(L, s);
      fill<uint32_t>(L, nb, nw, 0u, s);
      fill<U>(L, lab, nv, inf, s);
      L.go("init", k_set1<U>, 1, 1, s, lab, src, 0ull);
      L.go("init", k_set1<U>, 1, 1, s, snap, (int64_t)0, 0ull);
    };
    set_round(BmMin<3>{lab, nullptr, weighted ? g.w64.p : nullptr, snap, nb});
    P.finish = [=](Launcher &L, cudaStream_t s) {
      L.go("labels", k_labels_f64bits, grid_n(nv), 256, s, lab, nv, labels_d);
    };
  }
}

constexpr int64_t kPrTileBytes = 64ll << 20;  // rank-vector slice per source block
constexpr double kPrTileCoverage = 0.6;       // see prep_pr

void prep_pr(Program &P, Graph &g, const sg_params &p, RunBufs &rb, double *labels_d, int64_t thr,
             int64_t max_rounds, const Layout &lay) {
  const View &v = g.csc();
  const int64_t nv = v.nv;
  rb.alloc_common(nv, stats_cap(max_rounds));
  PullArgs a = rb.pull_args(v, thr, 0);
  a.vertex = p.sched == SG_SCHED_VERTEX;
  a.row_n = (uint32_t)nv;
  // devices > 1: CSC-row edge cut; pulls write only owned rows, so comm_sent
  // is 0 and every changed rank is broadcast to its mirrors (engine.py:88-113)
  const Cuts cuts = make_cuts(v, p.devices);
  uint32_t *mc = nullptr;
  if (p.devices > 1) mirror_counts(v, cuts, mc = P.buf<uint32_t>(nv));
  a.cuts = cuts;
  a.mcount = mc;
  int parts_nonempty = 0;
  for (int d = 0; d < cuts.D; ++d) parts_nonempty += cuts.c[d + 1] > cuts.c[d];
  double *inv = P.buf<double>(nv), *aux0 = P.buf<double>(nv), *aux1 = P.buf<double>(nv);
  unsigned long long *gmax = P.buf<unsigned long long>(1);
  const double d = p.damping, omd = 1.0 - p.damping;
  const int64_t *csr_off = g.csr.off.p;
  Ctl *ctl = rb.ctl.p;
  RoundStat *stats = rb.stats.p;
  uint32_t *largeq = rb.largeq.p, *hugeq = rb.hugeq.p;
  const int64_t *voff = v.off.p;
  const int64_t ne = v.ne;
  const double tol = p.tol;
  const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
  PrFold fold{aux0, aux1, aux1, aux0, labels_d, inv, d, omd, mc};

  // Source-block tiling: once the rank vector (V * 8 B) outgrows the L2, one
  // pull pass per source block gathers from an L2-resident slice (Tiles,
  // sg_graph.cu); rows carry their partial sums between passes (the blocks
  // are consecutive source ranges, i.e. consecutive stretches of every CSC
  // row, so the carried sum continues the reference's order).  Automatic
  // choice (p.reserved == 0): tile when the rank vector exceeds the slice AND
  // the graph's sources are not already skewed enough for the L2 to catch the
  // hot ranks by itself (rmat: the top quarter of vertices by out-degree
  // source most edges; tiling only adds row passes there).  A relabeled store
  // keeps its CSC rows in the reference's source order, which is not the
  // renamed id order the blocks cut, so it is never tiled.
  int64_t S = p.reserved > 0 ? (int64_t)p.reserved : 0;
  if (!S && nv * 8 > kPrTileBytes) {
    const int64_t B = (nv * 8 + kPrTileBytes - 1) / kPrTileBytes;
    const int64_t S0 = ((nv + B - 1) / B + 1023) / 1024 * 1024;
    if (g.source_coverage(S0) < kPrTileCoverage) S = S0;
  }
  if (lay.perm || p.devices != 1 || S >= nv) S = 0;
  const int64_t hs = exact_hs();
  const int nb = S > 0 ? (int)((nv + S - 1) / S) : 1;
  double *carry = nb > 1 ? P.buf<double>(nv) : nullptr;
  // heads[b]: block b's long-row tickets, heads[nb + b]: its SELL groups
  uint32_t *heads = P.buf<uint32_t>(2 * nb);
  long long *meta = P.buf<long long>(4);  // the reference's bins of the full CSC (round log)
  // SG_PR_SPLIT_ALL (experiments): every long row through the split path
  static const bool split_all = std::getenv("SG_PR_SPLIT_ALL") && std::atoi(std::getenv("SG_PR_SPLIT_ALL"));
  const int64_t split_min = split_all && thr != kNoHuge ? hs : std::max<int64_t>(thr, hs);
  std::vector<PrxArgs> xa((size_t)nb);
  for (int b = 0; b < nb; ++b) {
    const ExactLayout &L = nb > 1 ? g.tile_exact(S, hs, b) : g.exact(hs);
    const View &bv = nb > 1 ? g.tiles(S).blk[(size_t)b] : v;
    PrxArgs x = prx_args(bv, L, split_min, thr != kNoHuge, ctl, carry, gmax, heads + b,
                         [&](size_t bytes) { return (void *)P.buf<char>((int64_t)bytes); });
    x.cta_edges = rb.cta.p, x.cta_g = rb.cta_g, x.cta_rounds = rb.cta_rounds;
    xa[(size_t)b] = x;
  }
  const int gx = occupancy_grid(k_prx<0>, kTB);
  const int gbig = occupancy_grid(k_prx<1>, kTB), gsell = occupancy_grid(k_prx<2>, kTB);
  std::vector<PrxArgs> xs = xa;  // the SELL halves count their own tickets
  for (int b = 0; b < nb; ++b) xs[(size_t)b].head = heads + nb + b;
  // pass = the long rows (chunks, walkers, walked rows) then the SELL slices
  // split the pass when the long rows carry little of the work (uniform rmat25:
  // 106 -> 129 GTEPS); with skew they overlap the SELL slices inside one
  // launch and splitting them serialises the two (rmat24: 213 -> 173)
  static const int split_env = [] {
    const char *e = std::getenv("SG_PR_SPLIT");
    return e ? std::atoi(e) : -1;
  }();
  int64_t long_edges = 0, all_edges = 0;
  for (int b = 0; b < nb; ++b) {
    const ExactLayout &L = nb > 1 ? g.tile_exact(S, hs, b) : g.exact(hs);
    long_edges += L.big_edges, all_edges += L.big_edges + L.sell_edges;
  }
  const bool split_pass =
      split_env >= 0 ? split_env != 0 : long_edges * 4 < std::max<int64_t>(all_edges, 1);
  auto pass = [=](Launcher &L, cudaStream_t s, const char *name, int gain) {
    for (int b = 0; b < nb && !split_pass; ++b) {  // one launch over every ticket
      PrxArgs x = xa[(size_t)b];
      x.gain = gain;
      L.go(name, k_prx<0>, gx, kTB, s, x, fold);
    }
    for (int b = 0; b < nb && split_pass; ++b) {
      PrxArgs x = xa[(size_t)b], y = xs[(size_t)b];
      x.gain = y.gain = gain;
      if (x.nchunks + x.nsplit + x.nself) L.go(name, k_prx<1>, gbig, kTB, s, x, fold);
      if (y.ngroups) L.go(name, k_prx<2>, gsell, kTB, s, y, fold);
    }
  };
  P.init = [=](Launcher &L, cudaStream_t s) {
    L.go("init", k_ctl_init, 1, 1, s, ctl, 1, (uint32_t)nv);
    L.go("init", k_pr_init, grid_n(nv), 256, s, csr_off, nv, omd, inv, labels_d, aux0);
    L.go("init", k_copy_f64, grid_n(nv), 256, s, (const double *)aux0, nv, aux1);
    fill<unsigned long long>(L, gmax, 1, 0ull, s);
    fill<uint32_t>(L, heads, 2 * nb, 0u, s);
    // the reference's bins of the full CSC, for the round log (schedulers.py:144-167)
    L.go("init", k_static_bins, grid_n(nv), 256, s, voff, 0u, (uint32_t)nv, thr, largeq, hugeq,
         ctl, cuts);
    L.go("init", k_tile_store, 1, 1, s, ctl, meta);
    for (int b = 0; b < nb; ++b) {
      const PrxArgs &x = xa[(size_t)b];
      fill<uint32_t>(L, x.ck_meta, x.nchunks, 0u, s);
      if (x.nsplit) {
        L.go("init", k_prx_chunks, 1, 1024, s, x.off, x.big, x.nsplit, (uint32_t *)x.ck_first,
             (uint32_t *)x.ck_row);
        L.go("pr_guess", k_prx_guess_sums, grid_n((int64_t)x.nchunks * 32, kTB), kTB, s, x,
             (const double *)inv);
        L.go("pr_guess", k_prx_guess_scan, grid_n((int64_t)x.nsplit * 32, kTB), kTB, s, x);
      }
    }
    // eps_stop's gain (apps.py:163-171): one exact pass with aux = inv_outdeg
    if (ne) pass(L, s, "pr_gain", 1);
    fill<uint32_t>(L, heads, 2 * nb, 0u, s);
    for (int b = 0; b < nb; ++b) {  // round 0's binades (aux0 = (1-d) * inv_outdeg)
      const PrxArgs &x = xa[(size_t)b];
      if (x.nsplit) {
        L.go("pr_guess", k_prx_guess_sums, grid_n((int64_t)x.nchunks * 32, kTB), kTB, s, x,
             (const double *)aux0);
        L.go("pr_guess", k_prx_guess_scan, grid_n((int64_t)x.nsplit * 32, kTB), kTB, s, x);
      }
    }
  };
  PrStop stop{gmax, d, tol, ne, limit, max_rounds, cudaGraphConditionalHandle{}, 0, parts_nonempty};
  stop.bins = meta;
  if (a.vertex) {  // vertex scheduler (_kernels_py.py:88-97): one thread folds one row, in order
    PrOp op{aux0, aux1, aux1, aux0, labels_d, inv, d, omd};
    op.mcount = mc;
    double *hacc = P.buf<double>(1);
    P.round = [=](RoundCtx &c) {
      pull_round(c, a, op, false, hacc, false);
      PrStop st = stop;
      st.cond = c.cond, st.use_cond = c.use_cond;
      c.L.go("pr_finish", k_prx_finish, 1, 32, c.s, ctl, stats, (uint32_t)nv, st, cuts.D, heads,
             nb);
    };
  } else {
    P.round = [=](RoundCtx &c) {
      pass(c.L, c.s, "pr_pull", 0);
      PrStop st = stop;
      st.cond = c.cond, st.use_cond = c.use_cond;
      c.L.go("pr_finish", k_prx_finish, 1, 32, c.s, ctl, stats, (uint32_t)nv, st, cuts.D, heads,
             2 * nb);
    };
  }
  P.finish = [](Launcher &, cudaStream_t) {};
}

void prep_kcore(Program &P, Graph &g, const sg_params &p, RunBufs &rb, double *labels_d,
                int64_t thr, int64_t max_rounds, const Layout &lay) {
  const bool classic = (p.flags & SG_FLAG_TWC_CLASSIC) != 0;
  const View &v = g.sym();  // count rows: CSC(sym) and CSR(sym) rows hold the same multiset
  const int64_t nv = v.nv;
  rb.alloc_common(nv, stats_cap(max_rounds));
  rb.dying.alloc(std::max<int64_t>(nv, 1));
  PullArgs a = rb.pull_args(v, thr, 1);
  a.vertex = p.sched == SG_SCHED_VERTEX;
  // relabeled store: ids >= zsym are isolated; they die in round 0 (count 0 <
  // k, apps.py:220-225) with no neighbour to tell, so they are killed at init
  // and only counted in round 0's log (Ctl::fzero) -- the dense pass stops there
  const uint32_t rows = lay.zsym >= 0 && lay.zsym <= nv && p.devices == 1 && !a.vertex
                            ? (uint32_t)lay.zsym
                            : (uint32_t)nv;
  a.row_n = rows;
  const Cuts cuts = make_cuts(v, p.devices);  // sym CSC rows == sym CSR rows
  if (p.devices > 1) {
    uint32_t *mc = P.buf<uint32_t>(nv);
    mirror_counts(v, cuts, mc);
    a.mcount = mc;
  }
  a.cuts = cuts;
  PushArgs w = rb.push_args(v, kNoHuge);
  w.src_mode = 1;
  uint8_t *alive = P.buf<uint8_t>(nv);
  uint32_t *mark = P.buf<uint32_t>(nv), *hcnt = P.buf<uint32_t>(nv);
  Ctl *ctl = rb.ctl.p;
  P.init = [=](Launcher &L, cudaStream_t s) {
    L.go("init", k_ctl_init, 1, 1, s, ctl, 1, (uint32_t)nv);
    fill<uint8_t>(L, alive, nv, (uint8_t)1, s);
    if (rows < nv) {
      fill<uint8_t>(L, alive + rows, nv - rows, (uint8_t)0, s);
      L.go("init", k_set1<uint32_t>, 1, 1, s, &ctl->fzero, (int64_t)0, (uint32_t)(nv - rows));
    }
    fill<uint32_t>(L, mark, nv, 0u, s);
    fill<uint32_t>(L, hcnt, nv, 0u, s);
  };
  const KcOp op{alive, (uint32_t)std::min<int64_t>(p.k, 0xffffffffLL)};
  const OpMark mop{alive, mark};
  const bool blocked = p.blocked != 0;
  P.round = [=, &rb](RoundCtx &c) {
    pull_round(c, a, op, blocked, hcnt, classic);
    if (thr != kNoHuge)
      c.L.go("kcore_huge", k_pull_finish<KcOp, false>, 1, 1024, c.s, a, op, hcnt, PrStop{});
    c.L.go("kcore_kill", k_kcore_kill, grid_n(nv), 256, c.s, a, alive);
    c.L.go("kcore_stats", k_kcore_reset, 1, 1, c.s, a);
    c.L.go("mark_twc", k_push_twc<OpMark>, occupancy_grid(k_push_twc<OpMark>, kTB), kTB, c.s, w, mop);
    c.L.go("mark_large", k_push_large<OpMark>, occupancy_grid(k_push_large<OpMark>, kTB), kTB, c.s,
           w, mop);
    c.L.go("advance", k_kcore_advance, 1, 1, c.s, ctl, loop_of(rb, max_rounds, c));
  };
  P.finish = [=](Launcher &L, cudaStream_t s) {
    L.go("labels", k_labels_alive, grid_n(nv), 256, s, alive, nv, labels_d);
  };
}

// the device round log filled up before the run ended (see stats_cap)
struct CapError : Error {
  explicit CapError(const std::string &m) : Error(SG_ENOMEM, m) {}
};

struct RunResultC {
  int64_t rounds = 0;
  double ms = 0;
};

struct CtaOut {  // SG_FLAG_CTA_COUNTS results
  uint64_t *host = nullptr;
  int64_t rounds_cap = 0;
  int32_t *g = nullptr;
};

void run_app_on(Graph &g, const sg_params &p, double *labels_out, sg_round *rounds_out,
                int64_t cap, int64_t *nrounds, double *ms_out, Launcher *prof, const CtaOut *cta,
                const Layout &lay) {
  if (p.app < SG_APP_BFS || p.app > SG_APP_KCORE) throw Error(SG_ECONFIG, "unknown app");
  if (p.devices < 1) throw Error(SG_ECONFIG, "device count must be >= 1");
  if (g.nv > 0x7fffffffLL) throw Error(SG_ERANGE, "vertex ids must fit int32");
  if (g.is_part())
    throw Error(SG_ECONFIG, "an edge-cut partition runs with sg_team_run (one rank per GPU)");
  if ((p.app == SG_APP_BFS || p.app == SG_APP_SSSP) && (p.source < 0 || p.source >= g.nv))
    throw Error(SG_ECONFIG, "source " + std::to_string(p.source) + " outside graph");
  if (p.app == SG_APP_PR && !(p.damping > 0.0 && p.damping < 1.0))
    throw Error(SG_ECONFIG, "damping must be in (0, 1)");
  if (p.app == SG_APP_PR && !(p.tol > 0.0)) throw Error(SG_ECONFIG, "tolerance must be positive");
  if (p.app == SG_APP_KCORE && p.k < 1) throw Error(SG_ECONFIG, "k must be >= 1");
  if (p.app == SG_APP_SSSP && g.weighted && g.wmin < 0)
    throw Error(SG_ECONFIG, "sssp requires non-negative weights");
  const int64_t max_rounds =
      p.max_rounds > 0 ? p.max_rounds : 10 * std::max<int64_t>(g.nv, 1) + 256;
  if (p.sched < SG_SCHED_ALB || p.sched > SG_SCHED_EDGE) throw Error(SG_ECONFIG, "unknown scheduler");
  // alb: the resolved threshold; twc / vertex: no huge bin; lb / edge: every
  // active vertex goes through the prefix (the push engine runs dedicated
  // frontier-prefix / vertex / edge kernels, the pull and partitioned paths
  // the LB kernel with threshold 1 or a one-thread-per-row kernel)
  const int64_t thr = p.sched == SG_SCHED_TWC || p.sched == SG_SCHED_VERTEX ? kNoHuge
                      : p.sched == SG_SCHED_LB || p.sched == SG_SCHED_EDGE
                          ? 1
                          : std::max<int64_t>(1, p.threshold);
  *nrounds = 0;
  if (ms_out) *ms_out = 0.0;
  if (g.nv == 0) return;
  if (p.devices > 1 && !prof &&
      (p.app == SG_APP_BFS || p.app == SG_APP_SSSP || p.app == SG_APP_CC)) {
    // edge-cut partitions with label exchange (engine.py:64-113, 215-234)
    run_push_local_partitions(g, p, thr, max_rounds, labels_out, rounds_out, cap, nrounds,
                              ms_out);
    return;
  }
  // lazily built views (cached on the graph, like graph.py:102/117) are not timed
  if (p.app == SG_APP_CC || p.app == SG_APP_KCORE) g.sym();
  if (p.app == SG_APP_PR) g.csc();

  RunBufs rb;
  rb.want_cta = cta != nullptr;
  Program P;
  double *labels_d = P.buf<double>(g.nv);
  // the run's output -- float64 labels in the reference's numbering -- is
  // produced on the device inside the timed region; only the D2H is outside
  double *lab_out_d = lay.inv ? P.buf<double>(g.nv) : labels_d;
  P.inv = lay.inv, P.out = lab_out_d;
  switch (p.app) {
    case SG_APP_BFS:
    case SG_APP_SSSP:
    case SG_APP_CC: prep_push_min(P, g, p, rb, labels_d, thr, max_rounds, lay); break;
    case SG_APP_PR: prep_pr(P, g, p, rb, labels_d, thr, max_rounds, lay); break;
    case SG_APP_KCORE: prep_kcore(P, g, p, rb, labels_d, thr, max_rounds, lay); break;
  }
  cudaStream_t s;
  SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  Launcher plain;
  auto cleanup = [&] {
    cudaStreamSynchronize(s);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaStreamDestroy(s);
  };
  try {
    SG_CUDA(cudaEventCreate(&e0));
    SG_CUDA(cudaEventCreate(&e1));
    size_t body_nodes = 0;
    if (!prof) {
      // graph = WHILE(cond) { round }  — built before the timed region
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
      RoundCtx c{plain, s, cond, 1};
      P.round(c);
      SG_CUDA(cudaStreamEndCapture(s, &body));
      SG_CUDA(cudaGraphGetNodes(body, nullptr, &body_nodes));
      SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    }
    Launcher &L = prof ? *prof : plain;
    SG_CUDA(cudaEventRecord(e0, s));
    if (rb.cta.p)
      SG_CUDA(cudaMemsetAsync(rb.cta.p, 0, rb.cta.bytes(), s));
    P.init(L, s);
    int64_t rounds = 0;
    if (!prof) {
      SG_CUDA(cudaGraphLaunch(exec, s));
    } else {
      Ctl h;
      RoundCtx c{L, s, cudaGraphConditionalHandle{}, 0};
      const int64_t limit = std::min<int64_t>(max_rounds, rb.stats_cap);
      for (int64_t r = 0; r < limit; ++r) {
        P.round(c);
        SG_CUDA(cudaMemcpyAsync(&h, rb.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
        SG_CUDA(cudaStreamSynchronize(s));
        L.collect();
        if (h.done) break;
      }
    }
    P.finish(L, s);
    if (lay.inv && !P.unpermuted) L.go("labels", k_unpermute, grid_n(g.nv), 256, s, (const double *)labels_d, lay.inv,
                      g.nv, lab_out_d);
    SG_CUDA(cudaEventRecord(e1, s));
    SG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms_out) *ms_out = ms;
    Ctl h;
    SG_CUDA(cudaMemcpy(&h, rb.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
    rounds = h.round;
    if (!prof) g_launches.fetch_add((int64_t)body_nodes * rounds, std::memory_order_relaxed);
    if (prof) {
      SG_CUDA(cudaStreamSynchronize(s));
      L.collect();
    }
    std::vector<RoundStat> st((size_t)std::min<int64_t>(rounds, rb.stats_cap));
    if (!st.empty())
      SG_CUDA(cudaMemcpy(st.data(), rb.stats.p, sizeof(RoundStat) * st.size(),
                         cudaMemcpyDeviceToHost));
    if (rounds_out && !st.empty())
      std::memcpy(rounds_out, st.data(),
                  sizeof(RoundStat) * (size_t)std::min<int64_t>(cap, (int64_t)st.size()));
    *nrounds = rounds;
    SG_CUDA(cudaStreamSynchronize(s));
    if (cta && rb.cta.p) {
      *cta->g = (int32_t)rb.cta_g;
      const int64_t r = std::min<int64_t>({rounds, cta->rounds_cap, (int64_t)rb.cta_rounds});
      if (r > 0)
        SG_CUDA(cudaMemcpy(cta->host, rb.cta.p, sizeof(uint64_t) * rb.cta_g * r,
                           cudaMemcpyDeviceToHost));
    }
    if (labels_out)
      SG_CUDA(cudaMemcpy(labels_out, lab_out_d, sizeof(double) * g.nv, cudaMemcpyDeviceToHost));
    if (h.error == SG_ECONVERGE)
      throw Error(SG_ECONVERGE, "did not converge within " + std::to_string(max_rounds) + " rounds");
    if (h.error)
      throw CapError("round log capacity (" + std::to_string(rb.stats_cap) + ") exhausted");
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

// Hot-set size of the relabeled store (measured on rmat24, scripts/hotk_sweep.py):
// push apps gather labels of u32: the top 2^16 vertices (256 KB, about one
// SM's L1) first and the rest in id order is best (sssp +7 %, cc +7 %, bfs
// +4 %; a full degree order loses part of it again); pull apps (pr, kcore)
// gather over the whole vertex range every round and gain most from a full
// degree order (pr +15 %, kcore +16 %).  SG_HOT_K overrides (tuning runs).
int64_t hot_k(int64_t nv, int32_t app) {
  static const int64_t env = [] {
    const char *e = std::getenv("SG_HOT_K");
    return e ? std::atoll(e) : (int64_t)-1;
  }();
  const bool pull = app == SG_APP_PR || app == SG_APP_KCORE;
  const int64_t K = env >= 0 ? env : pull ? nv : (int64_t)1 << 16;
  return K > nv ? nv : K;
}

constexpr int64_t kRelabelMinV = (int64_t)1 << 20;

// Automatic choice: relabel skewed graphs of >= 2^20 vertices on one device,
// from the graph's second run on.  Building the relabeled store (degree sort +
// one renaming pass over the CSR: ~9 ms at rmat24, sg_graph.cu) costs more
// than one push run gains, so a graph that is created, run once and dropped
// (the e2e path) keeps its original numbering; resident graphs that are run
// again amortise it at once.  Without degree skew there is no hot set to
// cluster (uniform rmat25 pr: 120 -> 114 GTEPS relabeled), so graphs whose top
// 1 % of vertices source < 10 % of the edges keep their numbering.
constexpr double kRelabelMinSkew = 0.10;

// a relabeled store that does not fit next to what the device holds is not
// built (the run keeps the original numbering): free HBM after returning the
// allocator's cached blocks must exceed its size by 25 %
bool relabel_fits(Graph &g, bool in_first) {
  const int64_t need = g.relabel_bytes(in_first) + g.relabel_bytes(in_first) / 4;
  size_t fr = 0, tot = 0;
  SG_CUDA(cudaMemGetInfo(&fr, &tot));
  if ((int64_t)fr >= need) return true;
  dev_release_cached();
  SG_CUDA(cudaMemGetInfo(&fr, &tot));
  return (int64_t)fr >= need;
}

bool use_relabel(Graph &g, const sg_params &p) {
  if (p.devices != 1 || (p.flags & SG_FLAG_NO_RELABEL) || g.nv == 0) return false;
  const bool in_first = p.app == SG_APP_PR;
  if (p.flags & SG_FLAG_RELABEL) return relabel_fits(g, in_first);
  if (g.nv < kRelabelMinV || g.runs++ < 1) return false;
  return g.top1_share() >= kRelabelMinSkew && relabel_fits(g, in_first);
}

void run_app_layout(Graph &g, const sg_params &p, double *labels_out, sg_round *rounds_out,
                    int64_t cap, int64_t *nrounds, double *ms_out, Launcher *prof,
                    const CtaOut *cta);

void run_app(Graph &g, const sg_params &p, double *labels_out, sg_round *rounds_out, int64_t cap,
             int64_t *nrounds, double *ms_out, Launcher *prof, const CtaOut *cta = nullptr) {
  struct Restore {
    int64_t v = stats_cap_limit();
    ~Restore() { stats_cap_limit() = v; }
  } restore;
  try {
    run_app_layout(g, p, labels_out, rounds_out, cap, nrounds, ms_out, prof, cta);
  } catch (const CapError &) {  // a longer run than the first log holds: repeat with room
    const int64_t mr = p.max_rounds > 0 ? p.max_rounds : 10 * std::max<int64_t>(g.nv, 1) + 256;
    if (stats_cap_limit() >= std::min(mr, kStatsCapMax)) throw;
    stats_cap_limit() = std::min(mr, kStatsCapMax);
    run_app_layout(g, p, labels_out, rounds_out, cap, nrounds, ms_out, prof, cta);
  }
}

void run_app_layout(Graph &g, const sg_params &p, double *labels_out, sg_round *rounds_out,
                    int64_t cap, int64_t *nrounds, double *ms_out, Launcher *prof,
                    const CtaOut *cta) {
  if (!use_relabel(g, p)) {
    run_app_on(g, p, labels_out, rounds_out, cap, nrounds, ms_out, prof, cta, Layout{});
    return;
  }
  // the relabeled store is built once per graph (cached like csc / sym) and
  // is not timed; the source is renamed in, the labels renamed out
  // pr: vertices without in-edges last (their rows are skipped); kcore keeps
  // the plain degree order (in-edge-first measured 1.6 % slower there)
  Relabel &R = g.hot(hot_k(g.nv, p.app), p.app == SG_APP_PR);
  sg_params q = p;
  if ((p.app == SG_APP_BFS || p.app == SG_APP_SSSP) && p.source >= 0 && p.source < g.nv) {
    uint32_t s = 0;
    SG_CUDA(cudaMemcpy(&s, R.inv.p + p.source, sizeof(s), cudaMemcpyDeviceToHost));
    q.source = s;
  }
  Layout lay{R.perm.p, R.inv.p, R.zout, R.zsym, R.zin};
  if (p.app == SG_APP_CC && (lay.orig_src = maybe_sym_src(g))) lay.orig_sym = g.sym_.get();
  run_app_on(*R.g, q, labels_out, rounds_out, cap, nrounds, ms_out, prof, cta, lay);
}

}  // namespace
}  // namespace sg

// ====================================================================== C ABI
using sg::Error;

namespace sg {
namespace {
// Weight upload.  The host link (54.5 GB/s pinned, profiles/r2ay) bounds the
// e2e step and int64 weights are 2/3 of a weighted CSR's bytes: when every
// weight is in [0, 255] ([0, 65535]) host threads pack them into a pinned
// staging block -- while the offsets / targets are already in flight -- and
// 1/8 (1/4) of the bytes cross the link; the device widens them back to the
// int64 array the graph keeps.  Anything else goes up as int64.
template <class N>
__global__ void k_widen(const N *in, int64_t n, int64_t *out) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) out[i] = in[i];
}
// width 1 / 2: packed into `dst`; 0: some weight needs more than 16 bits
template <class N>
bool pack_weights(const int64_t *w, int64_t n, N *dst, int threads) {
  std::atomic<bool> ok{true};
  std::vector<std::thread> th;
  const int64_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t)
    th.emplace_back([&, t] {
      const int64_t a = t * per, b = std::min<int64_t>(n, a + per);
      uint64_t bad = 0;
      for (int64_t i = a; i < b; ++i) {
        const int64_t x = w[i];
        bad |= (uint64_t)x >> (8 * sizeof(N));  // negative or too wide
        dst[i] = (N)x;
      }
      if (bad) ok = false;
    });
  for (auto &x : th) x.join();
  return ok;
}
int g_last_weight_width = 8;  // bytes per weight of the last upload (sg_graph_last_upload)
void upload_weights(const int64_t *host, int64_t n, int64_t *dev, cudaStream_t s) {
  g_last_weight_width = 8;
  if (n <= 0) return;
  static const int cap = [] {  // SG_PACK_THREADS: host threads packing the weights
    const char *e = std::getenv("SG_PACK_THREADS");
    return e ? std::max(1, std::atoi(e)) : 16;
  }();
  // ranks of one node (torchrun's LOCAL_WORLD_SIZE) share the host's cores
  static const int local = [] {
    const char *e = std::getenv("LOCAL_WORLD_SIZE");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency() / (unsigned)local);
  const int threads = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)cap, (int64_t)hw, n >> 20}));
  // the weights' own stream: their slices cross the link beside the topology
  // still in flight on the caller's stream
  cudaStream_t ws = nullptr;
  SG_CUDA(cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking));
  struct WsGuard {
    cudaStream_t s;
    ~WsGuard() { cudaStreamSynchronize(s), cudaStreamDestroy(s); }
  } wsg{ws};
  (void)s;
  // one width at a time, packed in slices that are copied while the next one
  // is packed: up to 1 GB packed the whole array stays staged (8 slices, no
  // reuse); beyond, two alternating 256 MB pinned slots bound the host memory.
  // A weight too wide for the width abandons it (nothing of it is used).
  auto try_width = [&](auto zero) -> bool {
    using N = decltype(zero);
    // SG_PACK_WHOLE_MAX / SG_PACK_SLICE (bytes; tests): the staging bounds
    static const uint64_t whole_max = [] {
      const char *e = std::getenv("SG_PACK_WHOLE_MAX");
      return e ? (uint64_t)std::atoll(e) : ((uint64_t)1 << 30);
    }();
    static const int64_t slice_bytes = [] {
      const char *e = std::getenv("SG_PACK_SLICE");
      return e ? std::max<int64_t>(64, std::atoll(e)) : ((int64_t)256 << 20);
    }();
    const bool whole = sizeof(N) * (uint64_t)n <= whole_max;
    const int64_t slice = whole ? (n + 7) / 8 : std::max<int64_t>(1, slice_bytes / (int64_t)sizeof(N));
    DBuf<N> d((size_t)n);
    N *slot[2] = {(N *)host_alloc(sizeof(N) * (size_t)(whole ? n : slice)),
                  whole ? nullptr : (N *)host_alloc(sizeof(N) * (size_t)slice)};
    cudaEvent_t ev[2];
    SG_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    SG_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    bool ok = true;
    int k = 0;
    for (int64_t a0 = 0; a0 < n && ok; a0 += slice, k ^= 1) {
      const int64_t len = std::min<int64_t>(slice, n - a0);
      N *dst = whole ? slot[0] + a0 : slot[k];
      if (!whole && a0 >= 2 * slice) SG_CUDA(cudaEventSynchronize(ev[k]));  // slot k free again
      ok = pack_weights(host + a0, len, dst, threads);
      if (!ok) break;
      SG_CUDA(cudaMemcpyAsync(d.p + a0, dst, sizeof(N) * (size_t)len, cudaMemcpyHostToDevice, ws));
      SG_CUDA(cudaEventRecord(ev[k], ws));
    }
    if (ok) {
      k_widen<N><<<grid_n(n), 256, 0, ws>>>(d.p, n, dev);
      SG_CUDA(cudaGetLastError());
    }
    SG_CUDA(cudaStreamSynchronize(ws));  // slots and d are released below
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    host_free(slot[0]);
    if (slot[1]) host_free(slot[1]);
    return ok;
  };
  if (try_width(uint8_t{})) {
    g_last_weight_width = 1;
  } else if (try_width(uint16_t{})) {
    g_last_weight_width = 2;
  } else {
    SG_CUDA(cudaMemcpyAsync(dev, host, sizeof(int64_t) * n, cudaMemcpyHostToDevice, ws));
    SG_CUDA(cudaStreamSynchronize(ws));
  }
}
}  // namespace
}  // namespace sg

extern "C" {

const char *sg_last_error(void) { return sg::t_last_error.c_str(); }

int64_t sg_kernel_launches(void) { return sg::g_launches.load(); }

int sg_host_alloc(int64_t bytes, void **out) {
  return sg::guard([&] {
    if (bytes < 0) throw Error(SG_ECONFIG, "negative size");
    *out = sg::host_alloc((size_t)std::max<int64_t>(bytes, 1));
  });
}

void sg_host_free(void *p) {
  if (p) sg::host_free(p);
}

void sg_release_cached(void) { sg::dev_release_cached(); }

int sg_set_device(int32_t device) {
  return sg::guard([&] { SG_CUDA(cudaSetDevice(device)); });
}

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
    // the topology goes up asynchronously while host threads pack the weights
    cudaStream_t s = nullptr;
    SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamSynchronize(s), cudaStreamDestroy(s); }
    } sgd{s};
    SG_CUDA(cudaMemcpyAsync(g->csr.off.p, offsets, sizeof(int64_t) * (nv + 1),
                            cudaMemcpyHostToDevice, s));
    if (ne)
      SG_CUDA(cudaMemcpyAsync(g->csr.col.p, targets, sizeof(int32_t) * ne,
                              cudaMemcpyHostToDevice, s));
    if (weights) {
      g->w64.alloc(ne ? ne : 1);
      sg::upload_weights(weights, ne, g->w64.p, s);
      SG_CUDA(cudaStreamSynchronize(s));
      sg::weights_finalize(*g);
    } else {
      SG_CUDA(cudaStreamSynchronize(s));
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
    SG_CUDA(cudaDeviceSynchronize());
    sg::upload_weights(weights, src.ne, g->w64.p, nullptr);
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
    const sg::Graph &G = *g->g;
    *ne = which == 0 ? G.csr.ne : which == 1 ? (G.csc_ ? G.csc_->ne : G.ne)
                                             : (G.sym_ ? G.sym_->ne : 2 * G.ne);
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

int sg_graph_release_views(sg_graph *g) {
  return sg::guard([&] {
    if (!g) throw Error(SG_ECONFIG, "null graph");
    g->g->release_views();
  });
}

int sg_graph_build_ms(sg_graph *g, double out[4]) {
  return sg::guard([&] {
    if (!g) throw Error(SG_ECONFIG, "null graph");
    for (int i = 0; i < 4; ++i) out[i] = g->g->build_ms[i];
  });
}

void sg_graph_destroy(sg_graph *g) { delete g; }

int sg_run(sg_graph *g, const sg_params *p, double *labels_out, sg_round *rounds_out,
           int64_t rounds_cap, int64_t *nrounds, double *ms_out) {
  return sg::guard([&] {
    sg::run_app(*g->g, *p, labels_out, rounds_out, rounds_cap, nrounds, ms_out, nullptr);
  });
}

int sg_run_cta_counts(sg_graph *g, const sg_params *p, double *labels_out, sg_round *rounds_out,
                      int64_t rounds_cap, int64_t *nrounds, double *ms_out, uint64_t *cta_out,
                      int64_t cta_rounds_cap, int32_t *cta_g) {
  return sg::guard([&] {
    if (p->devices != 1) throw Error(SG_ECONFIG, "per-CTA counters need devices == 1");
    sg::CtaOut co{cta_out, cta_rounds_cap, cta_g};
    sg::run_app(*g->g, *p, labels_out, rounds_out, rounds_cap, nrounds, ms_out, nullptr, &co);
  });
}

int sg_run_profiled(sg_graph *g, const sg_params *p, double *labels_out, sg_round *rounds_out,
                    int64_t rounds_cap, int64_t *nrounds, double *ms_out, sg_kernel_time *kt,
                    int32_t kt_cap, int32_t *nkt) {
  return sg::guard([&] {
    sg::Launcher L;
    L.profile = true;
    *nkt = 0;
    auto report = [&] {
      int32_t n = 0;
      for (const auto &name : L.order) {
        if (n >= kt_cap) break;
        std::memset(kt[n].name, 0, sizeof(kt[n].name));
        std::strncpy(kt[n].name, name.c_str(), sizeof(kt[n].name) - 1);
        kt[n].launches = L.totals[name].first;
        kt[n].ms = L.totals[name].second;
        ++n;
      }
      *nkt = n;
    };
    try {
      sg::run_app(*g->g, *p, labels_out, rounds_out, rounds_cap, nrounds, ms_out, &L);
    } catch (...) {
      report();
      throw;
    }
    report();
  });
}

}  // extern "C"
