// sg_graph.cu — graph construction on the device.
//
// Every builder reproduces the reference's host construction bit for bit:
//   from_edges  = stable sort by source         (graph.py:63-76)
//   csc         = stable sort by target         (graph.py:95-113)
//   symmetrized = row v of CSR ++ row v of CSC  (graph.py:115-128: the stable sort of
//                 concat(src,dst) by source yields exactly that order)
//   generate_rmat / attach_random_weights: numpy PCG64 streams (graph.py:274-305)
// The LSD radix sort (CUB) is stable, which is what makes these identical.
#include <algorithm>
#include <chrono>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "sg_graph.cuh"

namespace sg {

namespace {

__global__ void k_offsets_from_sorted(const uint32_t *__restrict__ keys, int64_t ne, int64_t nv,
                                      int64_t *__restrict__ off) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= ne; i += stride) {
    int64_t hi = (i < ne) ? (int64_t)keys[i] : nv;        // rows [lo+1, hi] start at i
    int64_t lo = (i > 0) ? (int64_t)keys[i - 1] : -1;
    for (int64_t v = lo + 1; v <= hi; ++v) off[v] = i;
  }
}

// row id of every edge: one warp per row, coalesced writes
__global__ void k_expand_rows(const int64_t *__restrict__ off, int64_t nv,
                              uint32_t *__restrict__ rows) {
  int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nv; v += warps) {
    int64_t s = off[v], e = off[v + 1];
    for (int64_t i = s + lane_id(); i < e; i += 32) rows[i] = (uint32_t)v;
  }
}

__global__ void k_sym_offsets(const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                              int64_t nv, int64_t *__restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= nv; v += stride)
    out[v] = a[v] + b[v];
}

__global__ void k_sym_fill(const int64_t *__restrict__ aoff, const uint32_t *__restrict__ acol,
                           const int64_t *__restrict__ boff, const uint32_t *__restrict__ bcol,
                           const int64_t *__restrict__ soff, int64_t nv,
                           uint32_t *__restrict__ scol) {
  int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nv; v += warps) {
    int64_t o = soff[v];
    int64_t s = aoff[v], e = aoff[v + 1];
    for (int64_t i = s + lane_id(); i < e; i += 32) scol[o + (i - s)] = acol[i];
    o += e - s;
    s = boff[v], e = boff[v + 1];
    for (int64_t i = s + lane_id(); i < e; i += 32) scol[o + (i - s)] = bcol[i];
  }
}

// ---- numpy PCG64 (pcg_setseq_128_xsl_rr_64, step-then-output) -------------
typedef unsigned __int128 u128;
__host__ __device__ inline u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
}
__host__ __device__ inline uint64_t pcg_output(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned r = (unsigned)(s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}
// affine jump: state after `delta` steps is A*state + C
__host__ __device__ inline void pcg_jump(u128 inc, u128 delta, u128 &A, u128 &C) {
  u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
  while (delta) {
    if (delta & 1) { am *= cm; ap = ap * cm + cp; }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  A = am, C = ap;
}

constexpr int kRmatPer = 16;  // edges per thread (registers hold their src/dst bits)

// Level l, edge i uses draw l*E+i of the stream (graph.py:293-297):
// u = (next64 >> 11) * 2^-53;  q = searchsorted(cuts, u, 'right')
__global__ void __launch_bounds__(256) k_rmat(int scale, int64_t ne, uint64_t s_hi, uint64_t s_lo,
                                              uint64_t i_hi, uint64_t i_lo, uint64_t AE_hi,
                                              uint64_t AE_lo, uint64_t CE_hi, uint64_t CE_lo,
                                              double c0, double c1, double c2,
                                              uint32_t *__restrict__ src,
                                              uint32_t *__restrict__ dst) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i0 = t * kRmatPer;
  if (i0 >= ne) return;
  const u128 inc = ((u128)i_hi << 64) | i_lo;
  const u128 AE = ((u128)AE_hi << 64) | AE_lo, CE = ((u128)CE_hi << 64) | CE_lo;
  const u128 M = pcg_mult();
  u128 A, C;
  pcg_jump(inc, (u128)i0, A, C);
  u128 lvl = A * (((u128)s_hi << 64) | s_lo) + C;  // state before draw l*E + i0
  uint32_t s[kRmatPer], d[kRmatPer];
#pragma unroll
  for (int j = 0; j < kRmatPer; ++j) s[j] = 0, d[j] = 0;
  const int n = (int)min((int64_t)kRmatPer, ne - i0);
  for (int l = 0; l < scale; ++l) {
    u128 x = lvl;
#pragma unroll
    for (int j = 0; j < kRmatPer; ++j) {
      x = x * M + inc;
      double u = (double)(pcg_output(x) >> 11) * (1.0 / 9007199254740992.0);
      uint32_t q = (u >= c0) + (u >= c1) + (u >= c2);
      s[j] = (s[j] << 1) | (q >> 1);
      d[j] = (d[j] << 1) | (q & 1u);
    }
    lvl = AE * lvl + CE;
  }
#pragma unroll
  for (int j = 0; j < kRmatPer; ++j)
    if (j < n) src[i0 + j] = s[j], dst[i0 + j] = d[j];
}

// rng.integers(low, low + 2^j) with dtype int64 (graph.py:304): numpy's
// bounded path takes next_uint32 (low half of a 64-bit draw, then the high
// half) and Lemire-scales by 2^j: out = low + (u32 >> (32 - j)); no rejections.
__global__ void k_weights(int64_t ne, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                          int64_t low, int jbits, int64_t *__restrict__ w) {
  int64_t pair = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * pair >= ne) return;
  const u128 inc = ((u128)i_hi << 64) | i_lo;
  u128 A, C;
  pcg_jump(inc, (u128)pair + 1, A, C);
  uint64_t r = pcg_output(A * (((u128)s_hi << 64) | s_lo) + C);
  uint32_t lo = (uint32_t)r, hi = (uint32_t)(r >> 32);
  auto scale = [&](uint32_t u) -> int64_t {
    return low + (int64_t)(jbits == 0 ? 0 : (((uint64_t)u * (1ull << jbits)) >> 32));
  };
  w[2 * pair] = scale(lo);
  if (2 * pair + 1 < ne) w[2 * pair + 1] = scale(hi);
}

__global__ void k_fill_u32(uint32_t *__restrict__ p, int64_t n, uint32_t x) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = x;
}

__global__ void k_w32(const int64_t *__restrict__ w, int64_t ne, uint32_t *__restrict__ o) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += stride)
    o[i] = (uint32_t)w[i];
}

inline int grid_for(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  int64_t cap = (int64_t)sm_info().sms * 16;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) < n) ++b;
  return b;
}

}  // namespace

void build_csr_from_pairs(View &v, int64_t nv, uint32_t *src, uint32_t *dst, int64_t ne,
                          int key_bits) {
  v.nv = nv;
  v.ne = ne;
  v.off.alloc(nv + 1);
  v.col.alloc(ne ? ne : 1);
  DBuf<uint32_t> keys_out(ne ? ne : 1);
  if (ne) {
    size_t tmp = 0;
    SG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, src, keys_out.p, dst, v.col.p, ne, 0,
                                            key_bits));
    DBuf<char> t(tmp);
    SG_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, src, keys_out.p, dst, v.col.p, ne, 0,
                                            key_bits));
    g_launches.fetch_add(1);
  }
  SG_LAUNCH(k_offsets_from_sorted, grid_for(ne + 1), 256, 0, 0, keys_out.p, ne, nv, v.off.p);
  SG_CUDA(cudaDeviceSynchronize());
}

void build_transpose(View &out, const View &in) {
  DBuf<uint32_t> rows(in.ne ? in.ne : 1), keys(in.ne ? in.ne : 1);
  if (in.ne) {
    SG_LAUNCH(k_expand_rows, grid_for(in.nv * 32), 256, 0, 0, in.off.p, in.nv, rows.p);
    SG_CUDA(cudaMemcpy(keys.p, in.col.p, sizeof(uint32_t) * in.ne, cudaMemcpyDeviceToDevice));
  }
  build_csr_from_pairs(out, in.nv, keys.p, rows.p, in.ne, bits_for(in.nv));
}

void build_symmetrized(View &out, const View &csr, const View &csc) {
  out.nv = csr.nv;
  out.ne = csr.ne + csc.ne;
  out.off.alloc(out.nv + 1);
  out.col.alloc(out.ne ? out.ne : 1);
  SG_LAUNCH(k_sym_offsets, grid_for(out.nv + 1), 256, 0, 0, csr.off.p, csc.off.p, out.nv,
            out.off.p);
  SG_LAUNCH(k_sym_fill, grid_for(out.nv * 32), 256, 0, 0, csr.off.p, csr.col.p, csc.off.p,
            csc.col.p, out.off.p, out.nv, out.col.p);
  SG_CUDA(cudaDeviceSynchronize());
}

void rmat_pairs_device(int scale, int64_t ne, const uint64_t pcg[4], const double cuts[3],
                       uint32_t *src, uint32_t *dst) {
  u128 inc = ((u128)pcg[2] << 64) | pcg[3];
  u128 AE, CE;
  pcg_jump(inc, (u128)ne, AE, CE);
  int64_t threads = (ne + kRmatPer - 1) / kRmatPer;
  int64_t blocks = (threads + 255) / 256;
  SG_LAUNCH(k_rmat, (unsigned)blocks, 256, 0, 0, scale, ne, pcg[0], pcg[1], pcg[2], pcg[3],
            (uint64_t)(AE >> 64), (uint64_t)AE, (uint64_t)(CE >> 64), (uint64_t)CE, cuts[0],
            cuts[1], cuts[2], src, dst);
  SG_CUDA(cudaDeviceSynchronize());
}

void random_weights_device(int64_t ne, const uint64_t pcg[4], int64_t low, int j_bits,
                           int64_t *w64) {
  int64_t pairs = (ne + 1) / 2;
  if (!pairs) return;
  SG_LAUNCH(k_weights, (unsigned)((pairs + 255) / 256), 256, 0, 0, ne, pcg[0], pcg[1], pcg[2],
            pcg[3], low, j_bits, w64);
  SG_CUDA(cudaDeviceSynchronize());
}

void weights_finalize(Graph &g) {
  g.weighted = true;
  if (!g.ne) { g.wmin = g.wmax = 0; return; }
  DBuf<int64_t> mm(2);
  size_t tmp = 0;
  SG_CUDA(cub::DeviceReduce::Min(nullptr, tmp, g.w64.p, mm.p, g.ne));
  size_t tmp2 = 0;
  SG_CUDA(cub::DeviceReduce::Max(nullptr, tmp2, g.w64.p, mm.p + 1, g.ne));
  DBuf<char> t(std::max(tmp, tmp2));
  SG_CUDA(cub::DeviceReduce::Min(t.p, tmp, g.w64.p, mm.p, g.ne));
  SG_CUDA(cub::DeviceReduce::Max(t.p, tmp2, g.w64.p, mm.p + 1, g.ne));
  int64_t h[2];
  SG_CUDA(cudaMemcpy(h, mm.p, sizeof(h), cudaMemcpyDeviceToHost));
  g.wmin = h[0], g.wmax = h[1];
  if (g.wmin >= 0 && g.wmax < ((int64_t)1 << 32)) {
    g.w32.alloc(g.ne);
    SG_LAUNCH(k_w32, grid_for(g.ne), 256, 0, 0, g.w64.p, g.ne, g.w32.p);
    SG_CUDA(cudaDeviceSynchronize());
  }
}

namespace {
// lengths of row v's block-b segment: positions of the block bounds inside the
// (source-sorted) CSC row, by binary search
__global__ void k_tile_len(const int64_t *off, const uint32_t *col, int64_t nv, int64_t lo_id,
                           int64_t hi_id, int64_t *len) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st) {
    const int64_t b = off[v], e = off[v + 1];
    auto lower = [&](int64_t key) {  // first position with col >= key
      int64_t l = b, h = e;
      while (l < h) {
        const int64_t m = (l + h) >> 1;
        if ((int64_t)col[m] < key) l = m + 1;
        else h = m;
      }
      return l;
    };
    len[v] = lower(hi_id) - lower(lo_id);
  }
}
// copy row v's block segment into the block view (warp per row)
__global__ void k_tile_fill(const int64_t *off, const uint32_t *col, int64_t nv, int64_t lo_id,
                            const int64_t *boff, uint32_t *bcol) {
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nv; v += warps) {
    const int64_t b = off[v], e = off[v + 1], n = boff[v + 1] - boff[v];
    if (!n) continue;
    int64_t l = b, h = e;  // segment start: first col >= lo_id
    while (l < h) {
      const int64_t m = (l + h) >> 1;
      if ((int64_t)col[m] < lo_id) l = m + 1;
      else h = m;
    }
    for (int64_t j = lane; j < n; j += 32) bcol[boff[v] + j] = col[l + j];
  }
}
}  // namespace

namespace {
__global__ void k_outdeg(const int64_t *off, int64_t nv, uint32_t *deg) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st)
    deg[v] = (uint32_t)(off[v + 1] - off[v]);
}
}  // namespace

double Graph::source_coverage(int64_t K) {
  if (K == cov_k_) return cov_;
  cov_k_ = K;
  cov_ = 1.0;
  if (ne == 0 || K >= nv) return cov_;
  DBuf<uint32_t> deg(nv), sorted(nv);
  DBuf<unsigned long long> sum(1);
  SG_LAUNCH(k_outdeg, grid_for(nv), 256, 0, 0, csr.off.p, nv, deg.p);
  size_t t1 = 0, t2 = 0;
  SG_CUDA(cub::DeviceRadixSort::SortKeysDescending(nullptr, t1, deg.p, sorted.p, nv));
  SG_CUDA(cub::DeviceReduce::Sum(nullptr, t2, sorted.p, sum.p, K));
  DBuf<char> t(std::max(t1, t2));
  SG_CUDA(cub::DeviceRadixSort::SortKeysDescending(t.p, t1, deg.p, sorted.p, nv));
  SG_CUDA(cub::DeviceReduce::Sum(t.p, t2, sorted.p, sum.p, K));
  unsigned long long h = 0;
  SG_CUDA(cudaMemcpy(&h, sum.p, sizeof(h), cudaMemcpyDeviceToHost));
  cov_ = (double)h / (double)ne;
  return cov_;
}

double Graph::top1_share() {
  if (top1_ < 0.0) {
    const int64_t k_old = cov_k_;
    const double c_old = cov_;
    top1_ = source_coverage(std::max<int64_t>(1, nv / 100));
    cov_k_ = k_old, cov_ = c_old;  // keep the pr tiling's cached entry
  }
  return top1_;
}

const Tiles &Graph::tiles(int64_t S) {
  if (tiles_ && tiles_->S == S) return *tiles_;
  const View &c = csc();
  auto t = std::make_unique<Tiles>();
  t->S = S;
  const int64_t B = (nv + S - 1) / S;
  t->blk.resize((size_t)B);
  DBuf<int64_t> len(nv + 1);
  for (int64_t b = 0; b < B; ++b) {
    View &v = t->blk[(size_t)b];
    v.nv = nv;
    v.off.alloc(nv + 1);
    SG_LAUNCH(k_tile_len, grid_for(nv), 256, 0, 0, c.off.p, c.col.p, nv, b * S,
              std::min<int64_t>((b + 1) * S, nv), len.p);
    SG_CUDA(cudaMemset(len.p + nv, 0, sizeof(int64_t)));
    size_t tmp = 0;
    SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, len.p, v.off.p, nv + 1));
    DBuf<char> t2(tmp);
    SG_CUDA(cub::DeviceScan::ExclusiveSum(t2.p, tmp, len.p, v.off.p, nv + 1));
    SG_CUDA(cudaMemcpy(&v.ne, v.off.p + nv, sizeof(int64_t), cudaMemcpyDeviceToHost));
    v.col.alloc(v.ne ? v.ne : 1);
    SG_LAUNCH(k_tile_fill, grid_for(nv * 32), 256, 0, 0, c.off.p, c.col.p, nv, b * S, v.off.p,
              v.col.p);
    SG_CUDA(cudaDeviceSynchronize());
  }
  tiles_ = std::move(t);
  return *tiles_;
}

namespace {
__global__ void k_indeg(const uint32_t *__restrict__ col, int64_t ne, uint32_t *__restrict__ cnt) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += st)
    atomicAdd(cnt + col[i], 1u);
}
// key[v] = total degree (saturating), ids[v] = v
// key = total degree (saturating); in_first: 0 for vertices without in-edges
__global__ void k_degkey(const int64_t *__restrict__ off, const uint32_t *indeg, int64_t nv,
                         bool in_first, uint32_t *key, uint32_t *__restrict__ ids) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st) {
    const uint64_t d = (uint64_t)(off[v + 1] - off[v]) + indeg[v];
    key[v] = in_first && !indeg[v] ? 0u : (uint32_t)(d < 0xffffffffull ? d : 0xffffffffull);
    ids[v] = (uint32_t)v;
  }
}
// new id of the hot vertex of degree rank r: r itself, or -- spread, K a
// multiple of 32 -- line (r mod 32) x (K/32) + r / 32, so the 32 hottest
// vertices sit in 32 different 128-byte label lines (their reductions land on
// different L2 slices) while the hot set still packs 32 labels per line
__host__ __device__ __forceinline__ int64_t hot_pos(int64_t r, int64_t K, bool spread) {
  return spread ? (r & 31) * (K >> 5) + (r >> 5) : r;
}
__host__ __device__ __forceinline__ int64_t hot_rank(int64_t i, int64_t K, bool spread) {
  return spread ? (i % (K >> 5)) * 32 + i / (K >> 5) : i;
}
// the top-K (sorted) ids take [0, K); flag them
__global__ void k_hot_place(const uint32_t *__restrict__ sorted, int64_t K, bool spread,
                            uint32_t *__restrict__ perm, uint32_t *__restrict__ cold) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < K; r += st) {
    perm[hot_pos(r, K, spread)] = sorted[r];
    cold[sorted[r]] = 0u;
  }
}
// every other vertex after them, by class (1: out-degree > 0, 2: out 0 and
// in > 0, 3: isolated), each class in id order: new id = base[class] + rank
__global__ void k_cold_class(const int64_t *__restrict__ off, const uint32_t *__restrict__ indeg,
                             int64_t nv, uint32_t *__restrict__ cls) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st)
    if (cls[v]) cls[v] = off[v + 1] > off[v] ? 1u : indeg[v] ? 2u : 3u;
}
__global__ void k_count_nonzero(const uint32_t *__restrict__ x, int64_t n,
                                unsigned long long *__restrict__ out) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) c += x[i] != 0u;
  c = __reduce_add_sync(0xffffffffu, (unsigned)c);
  if ((threadIdx.x & 31u) == 0 && c) atomicAdd(out, c);
}
__global__ void k_class_flag(const uint32_t *__restrict__ cls, int64_t nv, uint32_t c,
                             uint32_t *__restrict__ flag) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st)
    flag[v] = cls[v] == c;
}
__global__ void k_cold_place(const uint32_t *__restrict__ cls, const uint32_t *__restrict__ rank,
                             int64_t nv, uint32_t c, int64_t base, uint32_t *__restrict__ perm) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += st)
    if (cls[v] == c) perm[base + rank[v]] = (uint32_t)v;
}
__global__ void k_invert(const uint32_t *__restrict__ perm, int64_t nv, uint32_t *__restrict__ inv) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += st)
    inv[perm[i]] = (uint32_t)i;
}
__global__ void k_perm_len(const int64_t *__restrict__ off, const uint32_t *__restrict__ perm,
                           int64_t nv, int64_t *__restrict__ len) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += st) {
    const uint32_t v = perm[i];
    len[i] = off[v + 1] - off[v];
  }
}
// new row i = old row perm[i] with its targets renamed (row order kept).
// Rows [0, nbig) -- the head of the hot prefix, i.e. the hubs -- are split
// over gridDim.y CTAs each (a 370 K-edge hub on one warp serialised the whole
// pass); the rest take one warp per row.
__global__ void k_perm_rows(const int64_t *__restrict__ off, const uint32_t *__restrict__ col,
                            const int64_t *__restrict__ w64, const uint32_t *__restrict__ w32,
                            const uint32_t *__restrict__ perm, const uint32_t *__restrict__ inv,
                            const int64_t *__restrict__ noff, int64_t nv, int64_t nbig,
                            int64_t K, bool spread, uint32_t *__restrict__ ncol,
                            int64_t *__restrict__ nw64, uint32_t *__restrict__ nw32) {
  auto copy = [&](int64_t i, int64_t j0, int64_t step) {
    const uint32_t v = perm[i];
    const int64_t s = off[v], n = off[v + 1] - s, o = noff[i];
    for (int64_t j = j0; j < n; j += step) {
      ncol[o + j] = inv[col[s + j]];
      if (nw64) nw64[o + j] = w64[s + j];
      if (nw32) nw32[o + j] = w32[s + j];
    }
  };
  if (gridDim.y > 1) {  // hub rows (degree ranks < nbig): CTA (x, y) takes rank x, stride over y
    if ((int64_t)blockIdx.x < nbig)
      copy(hot_pos(blockIdx.x, K, spread), (int64_t)blockIdx.y * blockDim.x + threadIdx.x,
           (int64_t)gridDim.y * blockDim.x);
    return;
  }
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nv; i += warps)
    if (i >= K || hot_rank(i, K, spread) >= nbig) copy(i, lane_id(), 32);
}
}  // namespace

int64_t Graph::relabel_bytes(bool in_first) const {
  int64_t b = (nv + 1) * 8 + ne * 4 + nv * 4 * 2;  // CSR copy + perm / inv
  b += nv * 4 * 5 + nv * 8;                         // build temporaries
  if (weighted) b += ne * 4;
  if (in_first) b += (nv + 1) * 8 + ne * 4;         // the permuted CSC
  else b += ne * 8;                                 // row sort: keys + weights out
  return b;
}

// src[e] = the row of edge e: one warp per row writes its id over the row
__global__ void k_row_ids(const int64_t *off, int64_t nv, uint32_t *src) {
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < nv; v += warps)
    for (int64_t e = off[v] + (threadIdx.x & 31); e < off[v + 1]; e += 32) src[e] = (uint32_t)v;
}

const uint32_t *Graph::sym_src() {
  if (!sym_src_.p) {
    const View &s = sym();
    DBuf<uint32_t> b((size_t)std::max<int64_t>(s.ne, 1));
    if (s.ne) SG_LAUNCH(k_row_ids, grid_for(s.nv * 32), 256, 0, 0, s.off.p, s.nv, b.p);
    SG_CUDA(cudaDeviceSynchronize());
    sym_src_ = std::move(b);
  }
  return sym_src_.p;
}

void Graph::release_views() {
  hot_.clear();
  sym_src_.release();
  if (is_part()) {  // a partition's view is its data, not a derived layout
    std::lock_guard<std::mutex> lk(exact_mu_);
    exact_.clear();
    dev_release_cached();
    return;
  }
  {
    std::lock_guard<std::mutex> lk(exact_mu_);
    exact_.clear();
  }
  tiles_.reset();
  sym_.reset();
  csc_.reset();
  cov_k_ = -1;
  top1_ = -1.0;
  dev_release_cached();
}

// batch boundaries of a row-sorted pass: rows [cut[k], cut[k+1]) hold about
// ne / nb edges (CUB's segmented sort counts items in int)
__global__ void k_row_batches(const int64_t *off, int64_t nv, int nb, int64_t *cut) {
  if (threadIdx.x || blockIdx.x) return;
  const int64_t E = off[nv];
  cut[0] = 0;
  for (int k = 1; k < nb; ++k) {
    const int64_t target = E / nb * k;
    int64_t lo = 0, hi = nv;  // first row r with off[r] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    cut[k] = lo > cut[k - 1] ? lo : cut[k - 1];
  }
  cut[nb] = nv;
}
// rebased segment bounds; rows of >= max_len edges become empty segments
// (left unsorted: a hub row's sorted targets are dense runs of ids, and 32
// lanes reducing into one bitmap word / label sector serialise at the L2)
__global__ void k_rebase(const int64_t *off, int64_t n, int64_t base, int64_t max_len, int *beg,
                         int *end) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += st) {
    const int64_t b = off[i] - base, e = off[i + 1] - base;
    beg[i] = (int)b;
    end[i] = e - b >= max_len ? (int)b : (int)e;
  }
}

// Sort every row of a push layout by target id (weights carried along).  The
// min-relaxation apps are indifferent to the order of a row's edges (BSP: the
// round's result is the min over all of them), and ascending targets let the
// lanes of one gather instruction share 32-byte label sectors where a row is
// dense -- in the relabeled store's hot set, where most edges of a skewed
// graph point.  Only the relabeled copy is sorted: the graph's own CSR keeps
// the caller's order (downloads, pr's summation order).
void sort_rows(View &v, DBuf<uint32_t> *w32) {
  if (v.ne <= 1 || v.nv == 0) return;
  const int64_t kMaxItems = (int64_t)1 << 30;
  const int nb = (int)((v.ne + kMaxItems - 1) / kMaxItems) + (v.ne > kMaxItems ? 1 : 0);
  DBuf<int64_t> cut(nb + 1);
  SG_LAUNCH(k_row_batches, 1, 1, 0, 0, v.off.p, v.nv, nb, cut.p);
  std::vector<int64_t> hc(nb + 1);
  SG_CUDA(cudaMemcpy(hc.data(), cut.p, sizeof(int64_t) * (nb + 1), cudaMemcpyDeviceToHost));
  std::vector<int64_t> ho(nb + 1);
  for (int k = 0; k <= nb; ++k)
    SG_CUDA(cudaMemcpy(&ho[k], v.off.p + hc[k], sizeof(int64_t), cudaMemcpyDeviceToHost));
  DBuf<uint32_t> kout(v.ne), vout(w32 ? v.ne : 0);
  // the unsorted (hub) rows keep their order: start from a copy
  SG_CUDA(cudaMemcpy(kout.p, v.col.p, sizeof(uint32_t) * v.ne, cudaMemcpyDeviceToDevice));
  if (w32) SG_CUDA(cudaMemcpy(vout.p, w32->p, sizeof(uint32_t) * v.ne, cudaMemcpyDeviceToDevice));
  const int64_t max_len = (int64_t)1 << 16;
  for (int k = 0; k < nb; ++k) {
    const int64_t r0 = hc[k], r1 = hc[k + 1], e0 = ho[k], n = ho[k + 1] - ho[k];
    if (r1 <= r0 || n <= 0) continue;
    if (n > 0x7fffffffLL) throw Error(SG_ERANGE, "row batch too large to sort");
    DBuf<int> rb(r1 - r0), re(r1 - r0);
    SG_LAUNCH(k_rebase, grid_for(r1 - r0 + 1), 256, 0, 0, v.off.p + r0, r1 - r0 + 1, e0, max_len,
              rb.p, re.p);
    size_t tb = 0;
    if (w32)
      SG_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, v.col.p + e0, kout.p + e0,
                                                  w32->p + e0, vout.p + e0, (int)n, (int)(r1 - r0),
                                                  rb.p, re.p));
    else
      SG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, v.col.p + e0, kout.p + e0, (int)n,
                                                 (int)(r1 - r0), rb.p, re.p));
    DBuf<char> t(std::max<size_t>(tb, 1));
    if (w32)
      SG_CUDA(cub::DeviceSegmentedSort::SortPairs(t.p, tb, v.col.p + e0, kout.p + e0,
                                                  w32->p + e0, vout.p + e0, (int)n, (int)(r1 - r0),
                                                  rb.p, re.p));
    else
      SG_CUDA(cub::DeviceSegmentedSort::SortKeys(t.p, tb, v.col.p + e0, kout.p + e0, (int)n,
                                                 (int)(r1 - r0), rb.p, re.p));
    g_launches.fetch_add(1);
    SG_CUDA(cudaDeviceSynchronize());
  }
  v.col = std::move(kout);
  if (w32) *w32 = std::move(vout);
}

Relabel &Graph::hot(int64_t K, bool in_first) {
  K = std::max<int64_t>(0, std::min(K, nv));
  const int64_t key = 2 * K + (in_first ? 1 : 0);
  auto it = hot_.find(key);
  if (it != hot_.end()) return *it->second;
  // one relabeled store at a time: each is a full copy of the CSR (plus its
  // own CSC / symmetrized views), so a graph run by push, pull and kcore apps
  // would otherwise hold several
  hot_.clear();
  const auto t_build = std::chrono::steady_clock::now();
  auto R = std::make_unique<Relabel>();
  R->K = K;
  R->in_first = in_first;
  R->perm.alloc(nv ? nv : 1);
  R->inv.alloc(nv ? nv : 1);
  auto h = std::make_unique<Graph>();
  h->nv = nv, h->ne = ne;
  h->csr.nv = nv, h->csr.ne = ne;
  h->csr.off.alloc(nv + 1);
  h->csr.col.alloc(ne ? ne : 1);
  if (nv) {
    // a indeg, e key then class, b ids then class rank, c sorted keys then
    // class flags, d sorted ids
    DBuf<uint32_t> a(nv), b(nv), c(nv), d(nv), e(nv);
    SG_CUDA(cudaMemset(a.p, 0, sizeof(uint32_t) * nv));
    if (ne) SG_LAUNCH(k_indeg, grid_for(ne), 256, 0, 0, csr.col.p, ne, a.p);
    SG_LAUNCH(k_degkey, grid_for(nv), 256, 0, 0, csr.off.p, a.p, nv, in_first, e.p, b.p);
    size_t t1 = 0, t2 = 0, t3 = 0;
    SG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, t1, e.p, c.p, b.p, d.p, nv));
    SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, c.p, b.p, nv));
    SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, (int64_t *)nullptr, (int64_t *)nullptr,
                                          nv + 1));
    DBuf<char> t(std::max({t1, t2, t3}));
    // stable: equal degrees keep ascending ids
    SG_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.p, t1, e.p, c.p, b.p, d.p, nv));
    g_launches.fetch_add(1);
    // vertices with any edge (keys sorted descending: the isolated ones are last)
    unsigned long long nonzero = 0;
    {
      DBuf<unsigned long long> cnt(1);
      SG_CUDA(cudaMemset(cnt.p, 0, sizeof(unsigned long long)));
      SG_LAUNCH(k_count_nonzero, grid_for(nv), 256, 0, 0, c.p, nv, cnt.p);
      SG_CUDA(cudaMemcpy(&nonzero, cnt.p, sizeof(nonzero), cudaMemcpyDeviceToHost));
    }
    SG_LAUNCH(k_fill_u32, grid_for(nv), 256, 0, 0, e.p, nv, 1u);
    static const bool spread_env = [] {
      const char *x = std::getenv("SG_HOT_SPREAD");
      return x ? std::atoi(x) != 0 : true;
    }();
    const bool spread = spread_env && K < nv && K % 32 == 0 && K >= 1024;
    if (K) SG_LAUNCH(k_hot_place, grid_for(K), 256, 0, 0, d.p, K, spread, R->perm.p, e.p);
    SG_LAUNCH(k_cold_class, grid_for(nv), 256, 0, 0, csr.off.p, a.p, nv, e.p);
    int64_t base = K;
    for (uint32_t cl = 1; cl <= 3; ++cl) {
      SG_LAUNCH(k_class_flag, grid_for(nv), 256, 0, 0, e.p, nv, cl, c.p);
      SG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, t2, c.p, b.p, nv));
      SG_LAUNCH(k_cold_place, grid_for(nv), 256, 0, 0, e.p, b.p, nv, cl, base, R->perm.p);
      uint32_t last_rank = 0, last_flag = 0;
      SG_CUDA(cudaMemcpy(&last_rank, b.p + nv - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost));
      SG_CUDA(cudaMemcpy(&last_flag, c.p + nv - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost));
      base += (int64_t)last_rank + last_flag;
      if (cl == 1) R->zout = base;
      if (cl == 2) R->zsym = base;
    }
    if (K == nv) {  // no cold region: the zero keys are numbered last
      R->zout = nv;
      R->zsym = in_first ? nv : (int64_t)nonzero;  // isolated vertices
      R->zin = in_first ? (int64_t)nonzero : -1;   // vertices without in-edges
    }
    SG_LAUNCH(k_invert, grid_for(nv), 256, 0, 0, R->perm.p, nv, R->inv.p);
    DBuf<int64_t> len(nv + 1);
    SG_LAUNCH(k_perm_len, grid_for(nv), 256, 0, 0, csr.off.p, R->perm.p, nv, len.p);
    SG_CUDA(cudaMemset(len.p + nv, 0, sizeof(int64_t)));
    SG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, t3, len.p, h->csr.off.p, nv + 1));
    // weights: the u32 copy the kernels stream, plus int64 only where a run
    // may need the float64-bit path (no u32 copy, or u32 path sums may overflow)
    const bool want64 =
        weighted && (!w32.p || (double)wmax * (double)std::max<int64_t>(nv - 1, 1) >= 4294967295.0);
    if (weighted) {
      h->weighted = true, h->wmin = wmin, h->wmax = wmax;
      if (w32.p) h->w32.alloc(ne ? ne : 1);
      h->w64.alloc(want64 && ne ? ne : 1);
    }
    const int64_t nbig = std::min<int64_t>(K, 4096);
    uint32_t *nw32 = weighted && w32.p ? h->w32.p : nullptr;
    int64_t *nw64 = want64 ? h->w64.p : nullptr;
    if (nbig)
      SG_LAUNCH(k_perm_rows, dim3((unsigned)nbig, 16), 256, 0, 0, csr.off.p, csr.col.p, w64.p,
                w32.p, R->perm.p, R->inv.p, h->csr.off.p, nv, nbig, K, spread, h->csr.col.p, nw64,
                nw32);
    SG_LAUNCH(k_perm_rows, grid_for(nv * 32), 256, 0, 0, csr.off.p, csr.col.p, w64.p, w32.p,
              R->perm.p, R->inv.p, h->csr.off.p, nv, nbig, K, spread, h->csr.col.p, nw64, nw32);
    SG_CUDA(cudaDeviceSynchronize());
    static const bool sort_env = [] {
      const char *x = std::getenv("SG_HOT_SORT");
      return x ? std::atoi(x) != 0 : true;
    }();
    // push layout only (pr's in-edge order is its summation order); the
    // int64-weight path is rare and keeps its order
    if (sort_env && !in_first && !want64) sort_rows(h->csr, nw32 ? &h->w32 : nullptr);
  } else {
    SG_CUDA(cudaMemset(h->csr.off.p, 0, sizeof(int64_t)));
    if (weighted) h->weighted = true, h->w64.alloc(1);
  }
  // pull layout (pr): the relabeled CSC is the original CSC with its rows
  // permuted and its sources renamed -- NOT the transpose of the relabeled
  // CSR, which would order every row by new source id.  The reference sums a
  // row in CSC order (ascending original source id, np.add.at), and with
  // floating point the order is the result (sg_prx.cuh).
  if (in_first && nv) {
    const View &c = csc();
    auto pv = std::make_unique<View>();
    pv->nv = nv, pv->ne = ne;
    pv->off.alloc(nv + 1);
    pv->col.alloc(ne ? ne : 1);
    DBuf<int64_t> len(nv + 1);
    SG_LAUNCH(k_perm_len, grid_for(nv), 256, 0, 0, c.off.p, R->perm.p, nv, len.p);
    SG_CUDA(cudaMemset(len.p + nv, 0, sizeof(int64_t)));
    size_t t4 = 0;
    SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t4, len.p, pv->off.p, nv + 1));
    DBuf<char> t(t4);
    SG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, t4, len.p, pv->off.p, nv + 1));
    const int64_t nbig = std::min<int64_t>(K, 4096);
    if (nbig)
      SG_LAUNCH(k_perm_rows, dim3((unsigned)nbig, 16), 256, 0, 0, c.off.p, c.col.p,
                (const int64_t *)nullptr, (const uint32_t *)nullptr, R->perm.p, R->inv.p,
                pv->off.p, nv, nbig, K, false, pv->col.p, (int64_t *)nullptr,
                (uint32_t *)nullptr);
    SG_LAUNCH(k_perm_rows, grid_for(nv * 32), 256, 0, 0, c.off.p, c.col.p,
              (const int64_t *)nullptr, (const uint32_t *)nullptr, R->perm.p, R->inv.p, pv->off.p,
              nv, nbig, K, false, pv->col.p, (int64_t *)nullptr, (uint32_t *)nullptr);
    SG_CUDA(cudaDeviceSynchronize());
    h->csc_ = std::move(pv);
  }
  R->g = std::move(h);
  Relabel &out = *R;
  hot_[key] = std::move(R);
  build_ms[2] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_build)
                    .count();
  return out;
}

const View &Graph::csc() {
  if (is_part() && !csc_)
    throw Error(SG_ECONFIG, "this edge-cut partition holds no CSC rows (partition kind " +
                                std::to_string(part.kind) + ")");
  if (!csc_) {
    const auto t0 = std::chrono::steady_clock::now();
    auto v = std::make_unique<View>();
    build_transpose(*v, csr);
    SG_CUDA(cudaDeviceSynchronize());
    csc_ = std::move(v);
    build_ms[0] =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return *csc_;
}

const View &Graph::sym() {
  if (is_part() && !sym_)
    throw Error(SG_ECONFIG, "this edge-cut partition holds no symmetrized rows (partition kind " +
                                std::to_string(part.kind) + ")");
  if (!sym_) {
    const View &c = csc();
    const auto t0 = std::chrono::steady_clock::now();
    auto v = std::make_unique<View>();
    build_symmetrized(*v, csr, c);
    SG_CUDA(cudaDeviceSynchronize());
    sym_ = std::move(v);
    build_ms[1] =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return *sym_;
}

}  // namespace sg
