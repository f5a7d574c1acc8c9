/*
 * sg_oracle.c — C restatement of the reference's ALB BSP path.
 * TEST INFRASTRUCTURE ONLY: linked by tests/, smoke() and bench.py's
 * cpu_baseline / --impl reference legs, never by the product library.
 *
 * Follows the reference simtgraph (/root/reference/pkg/src/simtgraph):
 *   per-edge operator     _kernels.pyx:48-64 (_apply_edge) / _kernels_py.py:69-85
 *   push-min fold         apps.py:67-74   (frontier = {v : merged < values}, ascending)
 *   bfs / sssp / cc init  apps.py:87-95, 108-111, 122-127
 *   pr                    apps.py:155-186 (inv_outdeg, eps_stop, new=(1-d)+d*acc)
 *   kcore                 apps.py:210-232 (count, dying, alive neighbours)
 *   BSP driver            engine.py:190-246 (snapshot values, out, max_rounds)
 * Scheduler choice does not change labels nor the per-round
 * (frontier_size, active_edges) log (verified against tests/golden), so this
 * restatement applies each frontier vertex's edges directly.  Pull sums are
 * accumulated per row in CSC edge order starting from 0.0 — exactly the order
 * the reference's alb (cyclic) / twc kernels produce with np.add.at — so pr
 * labels are bit-identical to the reference's alb/twc runs.
 *
 * nthreads > 1 parallelises over frontier vertices with OpenMP: min
 * reductions use a CAS loop (order-independent), pull rows stay sequential
 * per row, so results are identical for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { APP_BFS = 0, APP_SSSP = 1, APP_CC = 2, APP_PR = 3, APP_KCORE = 4 };
enum { SGO_OK = 0, SGO_ECONFIG = -1, SGO_ECONVERGE = -3, SGO_ENOMEM = -5 };

static inline void min_update(double *slot, double prop) {
  /* labels are >= 0 (or +inf): IEEE order == unsigned bit order */
  uint64_t want, cur = __atomic_load_n((uint64_t *)slot, __ATOMIC_RELAXED);
  memcpy(&want, &prop, 8);
  while (want < cur) {
    if (__atomic_compare_exchange_n((uint64_t *)slot, &cur, want, 1, __ATOMIC_RELAXED,
                                    __ATOMIC_RELAXED))
      break;
  }
}

static inline void min_update_serial(double *slot, double prop) {
  if (prop < *slot) *slot = prop; /* _kernels.pyx:63-64 */
}

/* Build the ascending list of v with a[v] < b[v]; returns count. */
static int64_t changed_list(int64_t nv, const double *merged, const double *values,
                            int64_t *out_ids) {
  int64_t n = 0;
  for (int64_t v = 0; v < nv; ++v)
    if (merged[v] < values[v]) out_ids[n++] = v;
  return n;
}

/*
 * voff/vtgt  traversal view (CSR for push apps, CSC for pr, sym CSR for kcore —
 *            for a symmetrized multigraph CSC and CSR rows hold the same multiset)
 * vw         float64 weights aligned with vtgt (sssp), may be NULL (unit weights)
 * goff/gtgt  the app graph CSR (pr: directed CSR for inv_outdeg / eps_stop;
 *            kcore: symmetrized CSR for the dying-neighbour walk)
 * round_log  cap x 2 int64: (frontier_size, active_edges) per round
 */
int sgo_run(int app, int64_t nv, const int64_t *voff, const int32_t *vtgt, const double *vw,
            const int64_t *goff, const int32_t *gtgt, int64_t source, int64_t k, double damping,
            double tol, int64_t max_rounds, int nthreads, double *labels, int64_t *round_log,
            int64_t cap, int64_t *nrounds) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  *nrounds = 0;
  if (max_rounds <= 0) max_rounds = 10 * (nv > 1 ? nv : 1) + 256; /* engine.py:199-202 */
  double *values = labels;
  double *out = (double *)malloc(sizeof(double) * (size_t)(nv ? nv : 1));
  int64_t *front = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nv ? nv : 1));
  int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nv ? nv : 1));
  double *inv = NULL, *aux = NULL;
  unsigned char *mark = NULL;
  if (!out || !front || !next) return SGO_ENOMEM;
  int64_t nf = 0;
  double eps_stop = 0.0, one_minus_d = 1.0 - damping;
  int push = (app == APP_BFS || app == APP_SSSP || app == APP_CC);

  switch (app) {
  case APP_BFS:
  case APP_SSSP:
    if (source < 0 || source >= nv) return SGO_ECONFIG; /* apps.py:89-90 */
    for (int64_t v = 0; v < nv; ++v) values[v] = INFINITY;
    values[source] = 0.0;
    front[0] = source;
    nf = 1;
    break;
  case APP_CC:
    for (int64_t v = 0; v < nv; ++v) values[v] = (double)v, front[v] = v;
    nf = nv;
    break;
  case APP_PR: {
    inv = (double *)calloc((size_t)(nv ? nv : 1), sizeof(double));
    aux = (double *)malloc(sizeof(double) * (size_t)(nv ? nv : 1));
    if (!inv || !aux) return SGO_ENOMEM;
    for (int64_t v = 0; v < nv; ++v) {
      int64_t d = goff[v + 1] - goff[v];
      if (d > 0) inv[v] = 1.0 / (double)d;
      values[v] = one_minus_d;
      front[v] = v;
    }
    nf = nv;
    /* gain[v] = sum over in-edges of inv_outdeg[src], CSR edge order
       (np.bincount, apps.py:166-168) == per-CSC-row sequential order */
    double worst = 0.0;
    if (voff[nv] > 0) {
      double gmax = 0.0;
      for (int64_t v = 0; v < nv; ++v) {
        double s = 0.0;
        for (int64_t e = voff[v]; e < voff[v + 1]; ++e) s += inv[vtgt[e]];
        if (v == 0 || s > gmax) gmax = s;
      }
      worst = damping * gmax;
    }
    eps_stop = tol / (worst > 1.0 ? worst : 1.0);
    break;
  }
  case APP_KCORE:
    mark = (unsigned char *)calloc((size_t)(nv ? nv : 1), 1);
    if (!mark) return SGO_ENOMEM;
    for (int64_t v = 0; v < nv; ++v) values[v] = 1.0, front[v] = v;
    nf = nv;
    break;
  default:
    return SGO_ECONFIG;
  }
  if (push) memcpy(out, values, sizeof(double) * (size_t)nv);

  int64_t rounds = 0;
  while (nf > 0) {
    if (rounds >= max_rounds) { *nrounds = rounds; free(out); free(front); free(next);
      free(inv); free(aux); free(mark); return SGO_ECONVERGE; }
    int64_t edges = 0;
    if (push) {
      /* out == values on entry (make_out copy, apps.py:55-56) */
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : edges) if (nthreads != 1)
      for (int64_t i = 0; i < nf; ++i) {
        int64_t u = front[i];
        double base = values[u];
        edges += voff[u + 1] - voff[u];
        for (int64_t e = voff[u]; e < voff[u + 1]; ++e) {
          double prop = app == APP_BFS ? base + 1.0
                        : app == APP_SSSP ? base + (vw ? vw[e] : 1.0)
                                          : base;
          if (nthreads == 1) min_update_serial(&out[vtgt[e]], prop);
          else min_update(&out[vtgt[e]], prop);
        }
      }
      int64_t nn = changed_list(nv, out, values, next);
      for (int64_t i = 0; i < nn; ++i) values[next[i]] = out[next[i]];
      int64_t *t = front; front = next; next = t;
      if (round_log && rounds < cap) round_log[2 * rounds] = nf, round_log[2 * rounds + 1] = edges;
      nf = nn;
    } else if (app == APP_PR) {
      for (int64_t v = 0; v < nv; ++v) aux[v] = values[v] * inv[v]; /* apps.py:176-177 */
      double delta = 0.0;
#pragma omp parallel for schedule(dynamic, 256) reduction(max : delta) reduction(+ : edges) if (nthreads != 1)
      for (int64_t v = 0; v < nv; ++v) {
        double acc = 0.0;
        for (int64_t e = voff[v]; e < voff[v + 1]; ++e) acc += aux[vtgt[e]];
        edges += voff[v + 1] - voff[v];
        volatile double scaled = damping * acc; /* two roundings, as numpy */
        double nw = one_minus_d + scaled;
        double dlt = fabs(nw - values[v]);
        if (dlt > delta) delta = dlt;
        out[v] = nw;
      }
      memcpy(values, out, sizeof(double) * (size_t)nv);
      if (round_log && rounds < cap) round_log[2 * rounds] = nf, round_log[2 * rounds + 1] = edges;
      nf = (delta <= eps_stop) ? 0 : nv; /* apps.py:181-186 */
    } else { /* kcore */
      int64_t ndying = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : edges) if (nthreads != 1)
      for (int64_t i = 0; i < nf; ++i) {
        int64_t v = front[i];
        double cnt = 0.0;
        for (int64_t e = voff[v]; e < voff[v + 1]; ++e) cnt += values[vtgt[e]];
        edges += voff[v + 1] - voff[v];
        out[v] = cnt;
      }
      for (int64_t i = 0; i < nf; ++i)
        if (out[front[i]] < (double)k) next[ndying++] = front[i];
      if (round_log && rounds < cap) round_log[2 * rounds] = nf, round_log[2 * rounds + 1] = edges;
      for (int64_t i = 0; i < ndying; ++i) values[next[i]] = 0.0; /* apps.py:225 */
      int64_t nn = 0;
      for (int64_t i = 0; i < ndying; ++i) {
        int64_t v = next[i];
        for (int64_t e = goff[v]; e < goff[v + 1]; ++e) {
          int32_t u = gtgt[e];
          if (!mark[u] && values[u] > 0.0) mark[u] = 1;
        }
      }
      for (int64_t u = 0; u < nv; ++u)
        if (mark[u]) { front[nn++] = u; mark[u] = 0; } /* np.unique -> ascending */
      nf = ndying ? nn : 0;
    }
    ++rounds;
  }
  *nrounds = rounds;
  free(out); free(front); free(next); free(inv); free(aux); free(mark);
  return SGO_OK;
}

/* Edge stream of generate_rmat (graph.py:274-298) on numpy's PCG64
 * (XSL-RR 128/64, step-then-output) — lets the CPU baseline build its graph
 * without numpy's single-threaded generator.  state/inc from
 * np.random.PCG64(seed).state; draw j = l*E + i for level l, edge i. */
typedef unsigned __int128 u128;
static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

static inline uint64_t pcg_out(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

static u128 pcg_advance(u128 state, u128 inc, u128 delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = inc;
  while (delta) {
    if (delta & 1) { acc_mult *= cur_mult; acc_plus = acc_plus * cur_mult + cur_plus; }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

void sgo_rmat_pairs(int scale, int64_t ne, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi,
                    uint64_t inc_lo, const double *cuts, int32_t *src, int32_t *dst,
                    int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  u128 s0 = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  const int64_t B = 1 << 16;
#pragma omp parallel for schedule(static)
  for (int64_t b0 = 0; b0 < ne; b0 += B) {
    int64_t b1 = b0 + B < ne ? b0 + B : ne;
    for (int64_t i = b0; i < b1; ++i) src[i] = dst[i] = 0;
    for (int l = 0; l < scale; ++l) {
      u128 s = pcg_advance(s0, inc, (u128)l * (u128)ne + (u128)b0);
      for (int64_t i = b0; i < b1; ++i) {
        s = s * PCG_MULT + inc;
        double u = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
        int q = (u >= cuts[0]) + (u >= cuts[1]) + (u >= cuts[2]); /* searchsorted right */
        src[i] = (src[i] << 1) | (q >> 1);
        dst[i] = (dst[i] << 1) | (q & 1);
      }
    }
  }
}

/* Graph.from_edges (graph.py:63-76): stable counting sort by source.
 * A sequential scatter in input order is stable by construction. */
void sgo_csr_from_pairs(int64_t ne, int64_t nv, const int32_t *src, const int32_t *dst,
                        const int64_t *w_in, int64_t *off, int32_t *tgt, int64_t *w_out) {
  memset(off, 0, sizeof(int64_t) * (size_t)(nv + 1));
  for (int64_t i = 0; i < ne; ++i) off[src[i] + 1]++;
  for (int64_t v = 0; v < nv; ++v) off[v + 1] += off[v];
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nv ? nv : 1));
  memcpy(cur, off, sizeof(int64_t) * (size_t)nv);
  for (int64_t i = 0; i < ne; ++i) {
    int64_t p = cur[src[i]]++;
    tgt[p] = dst[i];
    if (w_in) w_out[p] = w_in[i];
  }
  free(cur);
}

/* Graph.csc() (graph.py:95-113): stable transpose.  Row v of the result lists
 * the sources of v's in-edges in CSR edge order (a sequential scatter over
 * the CSR is the stable counting sort). */
void sgo_transpose(int64_t nv, const int64_t *off, const int32_t *tgt, int64_t *toff,
                   int32_t *ttgt) {
  int64_t ne = off[nv];
  memset(toff, 0, sizeof(int64_t) * (size_t)(nv + 1));
  for (int64_t e = 0; e < ne; ++e) toff[tgt[e] + 1]++;
  for (int64_t v = 0; v < nv; ++v) toff[v + 1] += toff[v];
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nv ? nv : 1));
  memcpy(cur, toff, sizeof(int64_t) * (size_t)nv);
  for (int64_t u = 0; u < nv; ++u)
    for (int64_t e = off[u]; e < off[u + 1]; ++e) ttgt[cur[tgt[e]]++] = (int32_t)u;
  free(cur);
}

/* Graph.symmetrized() (graph.py:115-128): from_edges(src ++ dst, dst ++ src)
 * stable-sorted by source gives row v = CSR row v ++ CSC row v. */
void sgo_symmetrize(int64_t nv, const int64_t *off, const int32_t *tgt, const int64_t *coff,
                    const int32_t *ctgt, int64_t *soff, int32_t *stgt, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  soff[0] = 0;
  for (int64_t v = 0; v < nv; ++v)
    soff[v + 1] = soff[v] + (off[v + 1] - off[v]) + (coff[v + 1] - coff[v]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < nv; ++v) {
    int64_t p = soff[v];
    for (int64_t e = off[v]; e < off[v + 1]; ++e) stgt[p++] = tgt[e];
    for (int64_t e = coff[v]; e < coff[v + 1]; ++e) stgt[p++] = ctgt[e];
  }
}
