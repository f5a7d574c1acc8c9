// sg_graph.cuh — the HBM-resident graph store (reference graph.py:29-177).
#pragma once
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "sg_common.cuh"

namespace sg {

// One traversal view: CSR rows (push) or CSC rows (pull), int64 offsets,
// u32 column ids (graph.py:33-34 dtypes; ids < 2^31 so u32 == int32 bits).
struct View {
  int64_t nv = 0, ne = 0;
  DBuf<int64_t> off;
  DBuf<uint32_t> col;
};

// The CSC split into B source blocks (pr, sg_engine.cu): block b holds, for
// every row, the in-edges whose source lies in [b*S, (b+1)*S) -- a contiguous
// sub-range of the CSC row, since CSC rows are sorted by source.  A pull pass
// over one block gathers from an S*8-byte slice of the rank vector that stays
// resident in L2 (the whole vector does not once V*8 B exceeds the L2).
struct ExactLayout;
struct Tiles {
  int64_t S = 0;
  std::vector<View> blk;
  // exact-order pr layouts of the blocks (built lazily, per Hs)
  int64_t ex_hs = 0;
  std::vector<std::unique_ptr<ExactLayout>> ex;
};

// Exact-order layout of a pull view for pr (sg_prx.cu).  The reference sums a
// row's in-edges one by one in CSC order starting from 0.0 (np.add.at applies
// them in array order, _kernels_py.py:73-75; the CSC keeps source order,
// graph.py:95-113), and with floating point that order IS the result.  So:
//  * rows with 1 <= deg < hs are stored sliced-ELL (SELL-32): slices of 32
//    rows (degree-sorted inside windows of 4096 consecutive rows), entry j of
//    the slice's lane l at scol[soff[s] + 32 j + l] -- one lane sums one row
//    left to right with fully coalesced adjacency loads;
//  * rows with deg >= hs (`big`, degree-descending) are summed in 256-edge
//    chunks whose exact sequential sum is formed in integer units of the
//    running sum's ulp (sg_prx.cuh).
// In a source block of a tiled CSC, a row's segment continues the row's sum:
// kFirst marks the first block holding edges of the row (start from 0.0),
// kLast the last one (fold the row); other blocks carry the partial sum.
struct ExactLayout {
  static constexpr uint8_t kFirst = 1, kLast = 2;
  static constexpr uint32_t kEmpty = 0xffffffffu;  // empty lane / padding entry
  int64_t hs = 0;
  int64_t rlo = 0, rhi = -1;  // the rows it covers
  int64_t nshort = 0, nslices = 0, sell_entries = 0, sell_edges = 0;
  DBuf<uint32_t> srow;   // [nslices * 32] row id (kEmpty: no row)
  DBuf<uint8_t> sflag;   // [nslices * 32] kFirst | kLast
  DBuf<int64_t> soff;    // [nslices + 1] slice start in scol
  DBuf<uint32_t> scol;   // [sell_entries]
  int64_t ngroups = 0;   // dynamic-fetch units: runs of consecutive slices of >= kGroupEntries
  DBuf<uint32_t> gfirst; // [ngroups + 1] first slice of each group
  static constexpr int64_t kGroupEntries = 256;
  int64_t nbig = 0, big_edges = 0;
  DBuf<uint32_t> big;    // [nbig] rows with deg >= hs, degree descending (ties by id)
  DBuf<uint8_t> bflag;   // [nbig]
  std::vector<int64_t> big_deg;  // host copy of their degrees (descending)
  double build_ms = 0;
};
// rows [rlo, rhi) of the view only (rhi < 0: all rows) -- one rank's edge-cut rows
void build_exact_layout(ExactLayout &L, const View &v, int64_t hs, const View &full, int64_t lo,
                        int64_t hi, int64_t rlo = 0, int64_t rhi = -1);

struct Relabel;

struct Graph {
  int64_t nv = 0, ne = 0;
  View csr;
  // Edge-cut partition (sg_peer.cu, Gluon's outgoing edge cut, engine.py:64-85):
  // this graph holds only rows [lo, hi) of one traversal view of a full graph
  // -- kind 0 the CSR (bfs / sssp, with the rows' weights), 1 the CSC (pr; csr
  // then keeps only the full CSR offsets, the out-degrees pr divides by),
  // 2 the symmetrized CSR (cc / kcore).  The view keeps V + 1 offsets (rows
  // outside the block are empty) so the single-device kernels index it by
  // global vertex id; its edges are the block's only.
  struct Part {
    int kind = -1;
    int rank = 0, world = 1;
    std::vector<long long> cuts;  // the reference's cuts of the full view (world + 1)
    int64_t lo = 0, hi = 0;
    int64_t full_ne = 0;          // edges of the full view
    std::shared_ptr<void> mirrors;  // the peer transport's mirror masks (sg_peer.cu)
    // block-local hot-vertex relabeling (sg_peer.cu): every block [c[k], c[k+1])
    // is renumbered onto itself in descending total degree, so the cuts,
    // owners, mirror sets and comm counters are the reference's; perm: new ->
    // old id, inv: old -> new (all V vertices, every rank holds both)
    bool relabeled = false;
    DBuf<uint32_t> perm, inv;
    // push / symmetrized relabel: the block's vertices without rows in the
    // view are numbered last, [zlo, hi) -- the compaction counts them instead
    // of queueing them (as the single-device store's edgeless tail)
    int64_t zlo = -1;
  } part;
  bool is_part() const { return part.kind >= 0; }
  bool weighted = false;
  int64_t wmin = 0, wmax = 0;
  DBuf<int64_t> w64;  // the reference's int64 weights (graph.py:35-37)
  DBuf<uint32_t> w32; // compact copy used by the sssp kernels when 0 <= w < 2^32
  std::unique_ptr<View> csc_;  // Graph.csc()         (graph.py:95-113), built lazily
  std::unique_ptr<View> sym_;  // Graph.symmetrized() (graph.py:115-128), built lazily
  // row id of every symmetrized edge (cc's streaming round 0), built lazily
  DBuf<uint32_t> sym_src_;
  const uint32_t *sym_src();
  const View &csc();
  const View &sym();
  std::unique_ptr<Tiles> tiles_;  // pr source blocks of the CSC, built lazily per S
  const Tiles &tiles(int64_t S);
  // exact-order pr layout of the CSC (and of the tiles' blocks), lazily per hs
  // (keyed by hs and the row range: ranks-as-threads runs build theirs concurrently)
  std::map<std::tuple<int64_t, int64_t, int64_t>, std::unique_ptr<ExactLayout>> exact_;
  std::mutex exact_mu_;
  const ExactLayout &exact(int64_t hs, int64_t rlo = 0, int64_t rhi = -1);
  const ExactLayout &tile_exact(int64_t S, int64_t hs, int64_t b);
  // fraction of the edges whose source is among the K highest out-degree
  // vertices (cached per K): how much of a pull's gather traffic a cache of K
  // rank values absorbs on its own
  double source_coverage(int64_t K);
  int64_t cov_k_ = -1;
  double cov_ = 0.0;
  // hot-vertex relabelings of this graph (built lazily, cached per K; see Relabel)
  std::map<int64_t, std::unique_ptr<Relabel>> hot_;
  Relabel &hot(int64_t K, bool in_first = false);
  int64_t runs = 0;  // single-device runs on this graph (the relabeling is built from the 2nd)
  // last build times (ms) of the derived layouts: csc, sym, relabeled store, exact pr
  double build_ms[4] = {0, 0, 0, 0};
  // HBM a relabeled store of this graph needs (estimate, bytes)
  int64_t relabel_bytes(bool in_first) const;
  void release_views();
  // share of the edges leaving the top 1 % of vertices by out-degree (cached;
  // rmat skewed: ~0.5, uniform: ~0.03) -- whether a degree relabeling pays
  double top1_share();
  double top1_ = -1.0;
};

// Hot-vertex relabeling: the kernel-side layout of the store.  The K vertices
// of highest total degree (out + in; ties by id) take ids [0, K) in
// descending-degree order and every other vertex keeps its relative order
// after them.  Their labels then share cache lines, so one SM's L1 holds the
// labels most random accesses hit (a scattered 4-byte gather that misses L1 is
// one L1->L2 request; the request path is what bounds the push kernels, ncu).
// The same permutation serves every view: total degree is the row length of
// the symmetrized graph, and the CSC / sym of the relabeled CSR are built from
// it.  Labels are invariant under renaming (BSP rounds touch the same vertex
// sets), so runs map the source in and the labels back out (sg_engine.cu).
struct Relabel {
  int64_t K = 0;
  // the cold vertices are numbered [out-degree > 0][out 0, in > 0][isolated],
  // each in id order: ids >= zout have no out-edges (CSR), ids >= zsym none in
  // the symmetrized graph either (their frontier members are only counted)
  int64_t zout = 0, zsym = 0;
  // in_first (the pull layouts): vertices without in-edges are numbered last,
  // from zin on -- a pull row with no in-edges keeps its initial value
  bool in_first = false;
  int64_t zin = -1;
  DBuf<uint32_t> perm;       // new id -> old id
  DBuf<uint32_t> inv;        // old id -> new id
  std::unique_ptr<Graph> g;  // the relabeled CSR (+ weights, w32)
};

// builders (sg_graph.cu)
// sort every row of a push layout by target id, u32 weights carried (sg_graph.cu)
void sort_rows(View &v, DBuf<uint32_t> *w32);
void build_csr_from_pairs(View &v, int64_t nv, uint32_t *src, uint32_t *dst, int64_t ne,
                          int key_bits);
void build_transpose(View &out, const View &in);
void build_symmetrized(View &out, const View &csr, const View &csc);
void rmat_pairs_device(int scale, int64_t ne, const uint64_t pcg[4], const double cuts[3],
                       uint32_t *src, uint32_t *dst);
void random_weights_device(int64_t ne, const uint64_t pcg[4], int64_t low, int j_bits,
                           int64_t *w64);
void weights_finalize(Graph &g);  // wmin / wmax / w32 from w64

// edge-cut partitioned push apps, D partitions on this GPU (sg_dist.cu)
void run_push_local_partitions(Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds,
                               double *labels_out, sg_round *rounds_out, int64_t cap,
                               int64_t *nrounds, double *ms_out);

}  // namespace sg

struct sg_graph {
  std::shared_ptr<sg::Graph> g;
};
