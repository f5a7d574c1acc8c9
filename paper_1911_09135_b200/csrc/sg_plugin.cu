// sg_plugin.cu — the reference's kernel-backend protocol on the device.
//
// sg_lb_kernel / sg_twc_kernel / sg_vertex_kernel / sg_edge_kernel implement
// _kernels_py.lb_kernel / twc_kernel / vertex_kernel / edge_kernel
// (_kernels_py.py:88-201) on caller-owned host buffers, including the modeled
// counters (per_cta_edges attribution, per-warp search paths, search accesses).
//   * push opcodes (min): order-free -> one thread per edge, atomicMin on an
//     order-preserving u64 key of the float64 label;
//   * OP_PULL_ADD: np.add.at applies additions in array order, i.e. per row in
//     edge order (blocked LB: pass-major order) starting from out[row]; one
//     thread per row replays exactly that order -> bit-identical float sums.
//     Row lists must therefore be duplicate-free (the engine's frontiers are).
#include <cmath>
#include <vector>

#include "sg_common.cuh"

namespace sg {
namespace {

constexpr int OP_BFS = 0, OP_SSSP = 1, OP_PULL_ADD = 3;  // OP_CC = 2: prop = value

__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void k_to_keys(double *out, int64_t n) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    unsigned long long k = dkey(out[i]);
    reinterpret_cast<unsigned long long *>(out)[i] = k;
  }
}
__global__ void k_from_keys(double *out, int64_t n) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    out[i] = dval(reinterpret_cast<unsigned long long *>(out)[i]);
}

struct PlugGraph {
  const int64_t *off;
  const int32_t *tgt;
  const double *w;  // may be empty (nw == 0)
  int64_t nw;
  const double *values, *aux;
  double *out;  // keys for push opcodes
  int opcode;
};

__device__ __forceinline__ void push_edge(const PlugGraph &g, int64_t row, int64_t e) {
  int32_t dst = g.tgt[e];
  double base = g.values[row];
  double prop = g.opcode == OP_BFS ? __dadd_rn(base, 1.0)
                : g.opcode == OP_SSSP ? __dadd_rn(base, g.w[e])
                                      : base;
  atomicMin(reinterpret_cast<unsigned long long *>(g.out) + dst, dkey(prop));
}

// the bisection of _kernels.pyx:67-77, returning the probe count too
__device__ __forceinline__ int64_t search(const int64_t *cum, int64_t n, int64_t g, int *probes) {
  int64_t lo = 0, hi = n - 1;
  int c = 0;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    ++c;
    if (g < cum[mid]) hi = mid;
    else lo = mid + 1;
  }
  *probes = c;
  return lo;
}

// ---- lb_kernel --------------------------------------------------------------
__global__ void k_lb_push(PlugGraph g, const int64_t *huge, const int64_t *cum, int64_t nh,
                          int64_t e) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < e; x += st) {
    int pr;
    int64_t o = search(cum, nh, x, &pr);
    int64_t row = huge[o];
    push_edge(g, row, g.off[row] + (x - (o ? cum[o - 1] : 0)));
  }
}

// one thread per owner segment, additions in the reference's array order
__global__ void k_lb_pull(PlugGraph g, const int64_t *huge, const int64_t *cum, int64_t nh,
                          int blocked, int64_t chunk) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < nh; o += st) {
    int64_t a = o ? cum[o - 1] : 0, b = cum[o];
    int64_t row = huge[o], base = g.off[row] - a;
    double acc = g.out[row];
    if (!blocked) {
      for (int64_t x = a; x < b; ++x) acc = __dadd_rn(acc, g.aux[g.tgt[base + x]]);
    } else {  // array order is (pass p, thread tid) with x = tid*chunk + p
      for (int64_t p = 0; p < chunk; ++p) {
        int64_t t0 = (a - p + chunk - 1) / chunk;
        if (a - p < 0) t0 = 0;
        for (int64_t t = t0; t * chunk + p < b; ++t)
          acc = __dadd_rn(acc, g.aux[g.tgt[base + t * chunk + p]]);
      }
    }
    g.out[row] = acc;
  }
}

// search accounting: one thread per (pass, warp) group (_kernels_py.py:189-200)
__global__ void k_lb_counters(const int64_t *cum, int64_t nh, int64_t e, int blocked,
                              int64_t chunk, int64_t passes, int64_t T, int64_t nwarps, int W,
                              long long *pwp, unsigned long long *accesses) {
  int64_t groups = passes * nwarps;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += st) {
    int64_t p = gi / nwarps, w = gi % nwarps;
    int64_t prev = -1, distinct = 0;
    unsigned long long acc = 0;
    for (int lane = 0; lane < W; ++lane) {
      int64_t tid = w * W + lane;
      int64_t x = blocked ? tid * chunk + p : p * T + tid;
      if (x >= e) break;
      int pr;
      int64_t o = search(cum, nh, x, &pr);
      if (o != prev) {
        ++distinct;
        acc += (unsigned long long)pr;
        prev = o;
      }
    }
    if (distinct) {
      atomicMax(pwp + w, (long long)distinct);
      atomicAdd(accesses, acc);
    }
  }
}

// per-CTA edge counts of an index space [0, e) mapped to threads:
// cyclic tid = x % T; blocked / edge-kernel tid = x / chunk
__global__ void k_cta_counts(int64_t e, int64_t T, int tpb, int num_ctas, int blocked,
                             int64_t chunk, long long *pce) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= num_ctas) return;
  int64_t cnt = 0;
  if (!blocked) {
    int64_t full = e / T, rem = e % T;
    int64_t lo = (int64_t)c * tpb, hi = lo + tpb;
    cnt = full * tpb + std::max<int64_t>(0, std::min<int64_t>(hi, rem) - lo);
  } else {
    int64_t lo = (int64_t)c * tpb * chunk, hi = lo + (int64_t)tpb * chunk;
    cnt = std::max<int64_t>(0, std::min<int64_t>(hi, e) - lo);
  }
  pce[c] += cnt;
}

// ---- row lists (twc bins, vertex / edge kernels) ----------------------------
// attribution: 0 thread (i%T)/tpb, 1 warp (i%Nw)/(tpb/W), 2 cta i%num_ctas, 3 none
__global__ void k_rows(PlugGraph g, const int64_t *rows, int64_t n, int attr, int64_t T,
                       int64_t nwarps, int wpc, int num_ctas, int tpb, long long *pce) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    int64_t v = rows[i];
    int64_t s = g.off[v], e = g.off[v + 1];
    if (attr != 3 && e > s) {
      int64_t cta = attr == 0 ? (i % T) / tpb : attr == 1 ? (i % nwarps) / wpc : i % num_ctas;
      atomicAdd((unsigned long long *)(pce + cta), (unsigned long long)(e - s));
    }
    if (g.opcode == OP_PULL_ADD) {
      double acc = g.out[v];
      for (int64_t x = s; x < e; ++x) acc = __dadd_rn(acc, g.aux[g.tgt[x]]);
      g.out[v] = acc;
    } else {
      for (int64_t x = s; x < e; ++x) push_edge(g, v, x);
    }
  }
}

__global__ void k_deg_sum(const int64_t *off, const int64_t *rows, int64_t n,
                          unsigned long long *sum) {
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    s += (unsigned long long)(off[rows[i] + 1] - off[rows[i]]);
  s = warp_sum(s);
  if (lane_id() == 0 && s) atomicAdd(sum, s);
}

inline int gridn(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32));
}

// host-side RAII staging of the plugin call
struct Stage {
  DBuf<int64_t> off;
  DBuf<int32_t> tgt;
  DBuf<double> w, values, aux, out;
  PlugGraph g{};
  int64_t nv = 0;

  Stage(const int64_t *offsets, int64_t nv_, const int32_t *targets, int64_t ne,
        const double *weights, int64_t nw, const double *vals, double *outp, const double *auxp,
        int64_t naux, int opcode)
      : nv(nv_) {
    if (opcode < OP_BFS || opcode > OP_PULL_ADD)
      throw Error(SG_ECONFIG, "unknown opcode " + std::to_string(opcode));
    if (opcode == OP_SSSP && nw < ne) throw Error(SG_ECONFIG, "sssp needs per-edge weights");
    if (opcode == OP_PULL_ADD && naux < nv) throw Error(SG_ECONFIG, "pull needs aux[num_vertices]");
    off.alloc(nv + 1);
    tgt.alloc(std::max<int64_t>(ne, 1));
    w.alloc(std::max<int64_t>(nw, 1));
    values.alloc(std::max<int64_t>(nv, 1));
    out.alloc(std::max<int64_t>(nv, 1));
    aux.alloc(std::max<int64_t>(naux, 1));
    SG_CUDA(cudaMemcpy(off.p, offsets, 8 * (nv + 1), cudaMemcpyHostToDevice));
    if (ne) SG_CUDA(cudaMemcpy(tgt.p, targets, 4 * ne, cudaMemcpyHostToDevice));
    if (nw) SG_CUDA(cudaMemcpy(w.p, weights, 8 * nw, cudaMemcpyHostToDevice));
    if (nv) {
      SG_CUDA(cudaMemcpy(values.p, vals, 8 * nv, cudaMemcpyHostToDevice));
      SG_CUDA(cudaMemcpy(out.p, outp, 8 * nv, cudaMemcpyHostToDevice));
    }
    if (naux) SG_CUDA(cudaMemcpy(aux.p, auxp, 8 * naux, cudaMemcpyHostToDevice));
    g = PlugGraph{off.p, tgt.p, w.p, nw, values.p, aux.p, out.p, opcode};
    if (opcode != OP_PULL_ADD && nv) SG_LAUNCH(k_to_keys, gridn(nv), 256, 0, 0, out.p, nv);
  }
  void finish(double *outp) {
    if (g.opcode != OP_PULL_ADD && nv) SG_LAUNCH(k_from_keys, gridn(nv), 256, 0, 0, out.p, nv);
    SG_CUDA(cudaDeviceSynchronize());
    if (nv) SG_CUDA(cudaMemcpy(outp, out.p, 8 * nv, cudaMemcpyDeviceToHost));
  }
};

template <class T>
DBuf<T> upload(const T *h, int64_t n) {
  DBuf<T> d(std::max<int64_t>(n, 1));
  if (n) SG_CUDA(cudaMemcpy(d.p, h, sizeof(T) * n, cudaMemcpyHostToDevice));
  return d;
}

void check_geometry(int num_ctas, int tpb, int ws) {
  if (num_ctas < 1 || tpb < 1 || ws < 1 || tpb % ws)
    throw Error(SG_ECONFIG, "invalid launch geometry");
}

}  // namespace
}  // namespace sg

using sg::Error;

extern "C" {

int sg_lb_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                 const double *weights, int64_t nw, const int64_t *huge,
                 const int64_t *cumulative, int64_t nhuge, const double *values, double *out,
                 const double *aux, int64_t naux, int32_t opcode, int32_t blocked,
                 int32_t num_ctas, int32_t tpb, int32_t ws, int64_t *per_cta_edges,
                 int64_t *per_warp_paths, int64_t *accesses) {
  return sg::guard([&] {
    sg::check_geometry(num_ctas, tpb, ws);
    if (nhuge < 1) throw Error(SG_ECONFIG, "lb kernel requires a non-empty prefix");
    const int64_t e = cumulative[nhuge - 1];
    const int64_t T = (int64_t)num_ctas * tpb, nwarps = T / ws;
    const int64_t chunk = (e + T - 1) / T;  // == number of passes
    sg::Stage st(offsets, nv, targets, ne, weights, nw, values, out, aux, naux, opcode);
    auto dh = sg::upload(huge, nhuge);
    auto dc = sg::upload(cumulative, nhuge);
    auto pce = sg::upload(per_cta_edges, num_ctas);
    auto pwp = sg::upload(per_warp_paths, nwarps);
    sg::DBuf<unsigned long long> acc(1);
    SG_CUDA(cudaMemset(acc.p, 0, 8));
    if (e > 0) {
      if (opcode == sg::OP_PULL_ADD)
        SG_LAUNCH(sg::k_lb_pull, sg::gridn(nhuge), 256, 0, 0, st.g, dh.p, dc.p, nhuge, blocked,
                  chunk);
      else
        SG_LAUNCH(sg::k_lb_push, sg::gridn(e), 256, 0, 0, st.g, dh.p, dc.p, nhuge, e);
      SG_LAUNCH(sg::k_cta_counts, (num_ctas + 255) / 256, 256, 0, 0, e, T, tpb, num_ctas, blocked,
                chunk, (long long *)pce.p);
      SG_LAUNCH(sg::k_lb_counters, sg::gridn(chunk * nwarps), 256, 0, 0, dc.p, nhuge, e, blocked,
                chunk, chunk, T, nwarps, ws, (long long *)pwp.p, acc.p);
    }
    st.finish(out);
    SG_CUDA(cudaMemcpy(per_cta_edges, pce.p, 8 * num_ctas, cudaMemcpyDeviceToHost));
    SG_CUDA(cudaMemcpy(per_warp_paths, pwp.p, 8 * nwarps, cudaMemcpyDeviceToHost));
    unsigned long long a = 0;
    SG_CUDA(cudaMemcpy(&a, acc.p, 8, cudaMemcpyDeviceToHost));
    *accesses = (int64_t)a;
  });
}

int sg_twc_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                  const double *weights, int64_t nw, const int64_t *small, int64_t nsmall,
                  const int64_t *medium, int64_t nmedium, const int64_t *large, int64_t nlarge,
                  const double *values, double *out, const double *aux, int64_t naux,
                  int32_t opcode, int32_t num_ctas, int32_t tpb, int32_t ws,
                  int64_t *per_cta_edges) {
  return sg::guard([&] {
    sg::check_geometry(num_ctas, tpb, ws);
    const int64_t T = (int64_t)num_ctas * tpb, nwarps = T / ws;
    sg::Stage st(offsets, nv, targets, ne, weights, nw, values, out, aux, naux, opcode);
    auto pce = sg::upload(per_cta_edges, num_ctas);
    const int64_t *lists[3] = {small, medium, large};
    const int64_t ns[3] = {nsmall, nmedium, nlarge};
    for (int b = 0; b < 3; ++b) {
      if (!ns[b]) continue;
      auto d = sg::upload(lists[b], ns[b]);
      SG_LAUNCH(sg::k_rows, sg::gridn(ns[b]), 256, 0, 0, st.g, d.p, ns[b], b, T, nwarps,
                tpb / ws, num_ctas, tpb, (long long *)pce.p);
      SG_CUDA(cudaDeviceSynchronize());
    }
    st.finish(out);
    SG_CUDA(cudaMemcpy(per_cta_edges, pce.p, 8 * num_ctas, cudaMemcpyDeviceToHost));
  });
}

int sg_vertex_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                     const double *weights, int64_t nw, const int64_t *frontier, int64_t nf,
                     const double *values, double *out, const double *aux, int64_t naux,
                     int32_t opcode, int32_t num_ctas, int32_t tpb, int64_t *per_cta_edges) {
  return sg::guard([&] {
    sg::check_geometry(num_ctas, tpb, 1);
    const int64_t T = (int64_t)num_ctas * tpb;
    sg::Stage st(offsets, nv, targets, ne, weights, nw, values, out, aux, naux, opcode);
    auto pce = sg::upload(per_cta_edges, num_ctas);
    if (nf) {
      auto d = sg::upload(frontier, nf);
      SG_LAUNCH(sg::k_rows, sg::gridn(nf), 256, 0, 0, st.g, d.p, nf, 0, T, T, 1, num_ctas, tpb,
                (long long *)pce.p);
    }
    st.finish(out);
    SG_CUDA(cudaMemcpy(per_cta_edges, pce.p, 8 * num_ctas, cudaMemcpyDeviceToHost));
  });
}

int sg_edge_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                   const double *weights, int64_t nw, const int64_t *frontier, int64_t nf,
                   const double *values, double *out, const double *aux, int64_t naux,
                   int32_t opcode, int32_t num_ctas, int32_t tpb, int64_t *per_cta_edges) {
  return sg::guard([&] {
    sg::check_geometry(num_ctas, tpb, 1);
    const int64_t T = (int64_t)num_ctas * tpb;
    sg::Stage st(offsets, nv, targets, ne, weights, nw, values, out, aux, naux, opcode);
    auto pce = sg::upload(per_cta_edges, num_ctas);
    if (nf) {
      auto d = sg::upload(frontier, nf);
      sg::DBuf<unsigned long long> m(1);
      SG_CUDA(cudaMemset(m.p, 0, 8));
      SG_LAUNCH(sg::k_deg_sum, sg::gridn(nf), 256, 0, 0, st.off.p, d.p, nf, m.p);
      unsigned long long hm = 0;
      SG_CUDA(cudaMemcpy(&hm, m.p, 8, cudaMemcpyDeviceToHost));
      if (hm) {
        // contiguous chunks of ceil(m/T) edges per thread (_kernels_py.py:100-117)
        const int64_t chunk = ((int64_t)hm + T - 1) / T;
        SG_LAUNCH(sg::k_rows, sg::gridn(nf), 256, 0, 0, st.g, d.p, nf, 3, T, T, 1, num_ctas, tpb,
                  (long long *)pce.p);
        SG_LAUNCH(sg::k_cta_counts, (num_ctas + 255) / 256, 256, 0, 0, (int64_t)hm, T, tpb,
                  num_ctas, 1, chunk, (long long *)pce.p);
      }
    }
    st.finish(out);
    SG_CUDA(cudaMemcpy(per_cta_edges, pce.p, 8 * num_ctas, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
