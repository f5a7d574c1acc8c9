// sg_prx.cu — the exact-order pull layout for pr (see ExactLayout, sg_graph.cuh).
//
// Built once per CSC (or per source block of a tiled CSC) and cached on the
// graph like csc() / sym(): a view of the graph, not part of a run.
//   short rows (1 <= deg < hs): sorted by (window of 4096 rows, degree
//     descending, id) and cut into slices of 32; each slice is stored
//     column-major (entry j of every lane, then entry j + 1), padded to the
//     slice's longest row with kEmpty.  The in-row order of the CSC is kept.
//   big rows (deg >= hs): listed by degree descending, ties by id.
#include <chrono>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "sg_graph.cuh"

namespace sg {
namespace {

constexpr int kWinBits = 12;   // rows per sorting window: 4096 (fold writes stay local)
constexpr int kDegBits = 13;   // hs <= 2^13
constexpr int kKeyBits = 31 - kWinBits + kDegBits + kWinBits;  // 44

inline int grid_of(int64_t n, int block = 256) {
  const int64_t g = (n + block - 1) / block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_info().sms * 32));
}

__device__ __forceinline__ void append64(bool p, unsigned long long k, unsigned long long *list,
                                         uint32_t *count) {
  const uint32_t m = __ballot_sync(kFull, p);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane_id() == (uint32_t)leader) base = atomicAdd(count, (uint32_t)__popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (p) list[base + __popc(m & lanemask_lt())] = k;
}

__global__ void k_ex_classify(const int64_t *__restrict__ off, int64_t rlo, int64_t rhi, int64_t hs,
                              unsigned long long *__restrict__ skeys, uint32_t *__restrict__ ns,
                              unsigned long long *__restrict__ bkeys, uint32_t *__restrict__ nb) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = rlo + (int64_t)blockIdx.x * blockDim.x; b < rhi; b += st) {
    const int64_t v = b + threadIdx.x;
    const int64_t d = v < rhi ? off[v + 1] - off[v] : 0;
    const bool sh = d >= 1 && d < hs, bg = d >= hs;
    const unsigned long long sk = ((unsigned long long)(v >> kWinBits) << (kDegBits + kWinBits)) |
                                  ((unsigned long long)(hs - 1 - d) << kWinBits) |
                                  (unsigned long long)(v & ((1 << kWinBits) - 1));
    append64(sh, sk, skeys, ns);
    append64(bg, ((unsigned long long)(0xffffffffu - (uint32_t)d) << 32) | (unsigned long long)v,
             bkeys, nb);
  }
}

__device__ __forceinline__ uint8_t row_flags(const int64_t *foff, const uint32_t *fcol, uint32_t v,
                                             int64_t lo, int64_t hi) {
  const int64_t a = foff[v], e = foff[v + 1];
  uint8_t f = 0;
  if ((int64_t)fcol[a] >= lo) f |= ExactLayout::kFirst;
  if ((int64_t)fcol[e - 1] < hi) f |= ExactLayout::kLast;
  return f;
}

__global__ void k_ex_slices(const unsigned long long *__restrict__ keys, int64_t n, int64_t hs,
                            const int64_t *__restrict__ foff, const uint32_t *__restrict__ fcol,
                            int64_t lo, int64_t hi, int64_t nslices, uint32_t *__restrict__ srow,
                            uint8_t *__restrict__ sflag, int64_t *__restrict__ slen) {
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += warps) {
    const int64_t i = s * 32 + lane_id();
    uint32_t v = ExactLayout::kEmpty, d = 0;
    uint8_t f = 0;
    if (i < n) {
      const unsigned long long k = keys[i];
      v = (uint32_t)(((k >> (kDegBits + kWinBits)) << kWinBits) | (k & ((1u << kWinBits) - 1)));
      d = (uint32_t)(hs - 1 - (int64_t)((k >> kWinBits) & ((1u << kDegBits) - 1)));
      f = row_flags(foff, fcol, v, lo, hi);
    }
    srow[i] = v;
    sflag[i] = f;
    const uint32_t len = __reduce_max_sync(kFull, d);
    if (lane_id() == 0) slen[s] = 32 * (int64_t)len;
  }
}

__global__ void k_ex_fill(const int64_t *__restrict__ off, const uint32_t *__restrict__ col,
                          const uint32_t *__restrict__ srow, const int64_t *__restrict__ soff,
                          int64_t nslices, uint32_t *__restrict__ scol) {
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += warps) {
    const uint32_t v = srow[s * 32 + lane_id()];
    const int64_t a = v != ExactLayout::kEmpty ? off[v] : 0;
    const int64_t d = v != ExactLayout::kEmpty ? off[v + 1] - a : 0;
    const int64_t o = soff[s], len = (soff[s + 1] - o) / 32;
    for (int64_t j = 0; j < len; ++j)
      scol[o + 32 * j + lane_id()] = j < d ? col[a + j] : ExactLayout::kEmpty;
  }
}

__global__ void k_ex_big(const unsigned long long *__restrict__ keys, int64_t n,
                         const int64_t *__restrict__ foff, const uint32_t *__restrict__ fcol,
                         int64_t lo, int64_t hi, uint32_t *__restrict__ big,
                         uint8_t *__restrict__ bflag, int64_t *__restrict__ bdeg) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    const unsigned long long k = keys[i];
    const uint32_t v = (uint32_t)k;
    big[i] = v;
    bflag[i] = row_flags(foff, fcol, v, lo, hi);
    bdeg[i] = (int64_t)(0xffffffffu - (uint32_t)(k >> 32));
  }
}

}  // namespace

void build_exact_layout(ExactLayout &L, const View &v, int64_t hs, const View &full, int64_t lo,
                        int64_t hi, int64_t rlo, int64_t rhi) {
  if (hs < 2 || hs > (1 << kDegBits)) throw Error(SG_ECONFIG, "exact layout: hs out of range");
  const auto t0 = std::chrono::steady_clock::now();
  L.hs = hs;
  const int64_t nv = v.nv;
  DBuf<unsigned long long> sk(std::max<int64_t>(nv, 1)), bk(std::max<int64_t>(nv, 1));
  DBuf<uint32_t> cnt(2);
  SG_CUDA(cudaMemset(cnt.p, 0, 2 * sizeof(uint32_t)));
  if (rhi < 0) rhi = nv;
  if (rhi > rlo)
    SG_LAUNCH(k_ex_classify, grid_of(rhi - rlo), 256, 0, 0, v.off.p, rlo, rhi, hs, sk.p, cnt.p,
              bk.p, cnt.p + 1);
  uint32_t h[2];
  SG_CUDA(cudaMemcpy(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost));
  L.nshort = h[0], L.nbig = h[1];
  // short rows
  DBuf<unsigned long long> sk2(std::max<int64_t>(L.nshort, 1));
  size_t tb = 0;
  if (L.nshort) {
    SG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, sk.p, sk2.p, (int)L.nshort, 0, kKeyBits));
    DBuf<char> t(tb);
    SG_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tb, sk.p, sk2.p, (int)L.nshort, 0, kKeyBits));
  }
  L.nslices = (L.nshort + 31) / 32;
  L.srow.alloc(std::max<int64_t>(L.nslices * 32, 1));
  L.sflag.alloc(std::max<int64_t>(L.nslices * 32, 1));
  L.soff.alloc(L.nslices + 1);
  {
    DBuf<int64_t> slen(L.nslices + 1);
    SG_CUDA(cudaMemset(slen.p + L.nslices, 0, sizeof(int64_t)));
    if (L.nslices)
      SG_LAUNCH(k_ex_slices, grid_of(L.nslices * 32), 256, 0, 0, sk2.p, L.nshort, hs, full.off.p,
                full.col.p, lo, hi, L.nslices, L.srow.p, L.sflag.p, slen.p);
    size_t ts = 0;
    SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, ts, slen.p, L.soff.p, L.nslices + 1));
    DBuf<char> t(ts);
    SG_CUDA(cub::DeviceScan::ExclusiveSum(t.p, ts, slen.p, L.soff.p, L.nslices + 1));
  }
  SG_CUDA(cudaMemcpy(&L.sell_entries, L.soff.p + L.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost));
  L.scol.alloc(std::max<int64_t>(L.sell_entries, 1));
  if (L.nslices)
    SG_LAUNCH(k_ex_fill, grid_of(L.nslices * 32), 256, 0, 0, v.off.p, v.col.p, L.srow.p, L.soff.p,
              L.nslices, L.scol.p);
  // fetch groups: consecutive slices until >= kGroupEntries entries (one
  // atomic per group instead of one per slice of a few short rows)
  {
    std::vector<int64_t> so((size_t)L.nslices + 1);
    SG_CUDA(cudaMemcpy(so.data(), L.soff.p, sizeof(int64_t) * so.size(), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> gf;
    for (int64_t s0 = 0; s0 < L.nslices;) {
      gf.push_back((uint32_t)s0);
      int64_t s1 = s0 + 1;
      while (s1 < L.nslices && so[(size_t)s1] - so[(size_t)s0] < ExactLayout::kGroupEntries) ++s1;
      s0 = s1;
    }
    gf.push_back((uint32_t)L.nslices);
    L.ngroups = (int64_t)gf.size() - 1;
    L.gfirst.alloc(gf.size());
    SG_CUDA(cudaMemcpy(L.gfirst.p, gf.data(), sizeof(uint32_t) * gf.size(), cudaMemcpyHostToDevice));
  }
  // big rows
  L.big.alloc(std::max<int64_t>(L.nbig, 1));
  L.bflag.alloc(std::max<int64_t>(L.nbig, 1));
  L.big_deg.assign((size_t)L.nbig, 0);
  if (L.nbig) {
    DBuf<unsigned long long> bk2(L.nbig);
    size_t tbb = 0;
    SG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tbb, bk.p, bk2.p, (int)L.nbig));
    DBuf<char> t(tbb);
    SG_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tbb, bk.p, bk2.p, (int)L.nbig));
    DBuf<int64_t> bd(L.nbig);
    SG_LAUNCH(k_ex_big, grid_of(L.nbig), 256, 0, 0, bk2.p, L.nbig, full.off.p, full.col.p, lo, hi,
              L.big.p, L.bflag.p, bd.p);
    SG_CUDA(cudaMemcpy(L.big_deg.data(), bd.p, sizeof(int64_t) * L.nbig, cudaMemcpyDeviceToHost));
  }
  L.big_edges = 0;
  for (int64_t d : L.big_deg) L.big_edges += d;
  L.sell_edges = v.ne - L.big_edges;
  SG_CUDA(cudaDeviceSynchronize());
  L.build_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

const ExactLayout &Graph::exact(int64_t hs, int64_t rlo, int64_t rhi) {
  if (rhi < 0) rhi = nv;
  std::lock_guard<std::mutex> lk(exact_mu_);
  auto &slot = exact_[std::make_tuple(hs, rlo, rhi)];
  if (!slot) {
    const View &c = csc();
    auto L = std::make_unique<ExactLayout>();
    build_exact_layout(*L, c, hs, c, 0, nv, rlo, rhi);
    L->rlo = rlo, L->rhi = rhi;
    build_ms[3] = L->build_ms;
    slot = std::move(L);
  }
  return *slot;
}

const ExactLayout &Graph::tile_exact(int64_t S, int64_t hs, int64_t b) {
  const Tiles &T0 = tiles(S);
  Tiles &T = *tiles_;
  (void)T0;
  if (T.ex_hs != hs || T.ex.size() != T.blk.size()) {
    T.ex.clear();
    T.ex.resize(T.blk.size());
    T.ex_hs = hs;
  }
  auto &slot = T.ex[(size_t)b];
  if (!slot) {
    auto L = std::make_unique<ExactLayout>();
    build_exact_layout(*L, T.blk[(size_t)b], hs, csc(), b * S, std::min<int64_t>((b + 1) * S, nv));
    slot = std::move(L);
  }
  return *slot;
}

}  // namespace sg
