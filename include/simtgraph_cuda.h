/*
 * simtgraph_cuda.h — C ABI of libsimtgraph_cuda.so, the B200 (sm_100a)
 * implementation of the reference simtgraph's ALB hot path.
 *
 * Two cuts, both taken from the reference's own interfaces:
 *
 *  1. Run level (the performance cut).  Replaces the body of
 *     engine.run / engine.run_app (/root/reference/pkg/src/simtgraph/
 *     engine.py:190-261): the whole BSP loop — inspection, huge-vertex LB
 *     kernel, TWC bins, push/pull operator, frontier fold, edge-cut label
 *     sync — runs on the device; the caller gets float64 labels (apps.py:63-64)
 *     and one sg_round per BSP round (engine.py:116-163 RoundRecord).
 *
 *  2. Kernel level (the reference's plugin seam, kernels.py:16-41).
 *     sg_lb_kernel / sg_twc_kernel / sg_vertex_kernel / sg_edge_kernel take
 *     exactly the buffers of _kernels_py.lb_kernel / twc_kernel /
 *     vertex_kernel / edge_kernel (_kernels_py.py:88-201): caller-owned host
 *     arrays, `out`, `per_cta_edges`, `per_warp_paths` mutated in place.
 *
 * Conventions: every function returns 0 on success or a negative SG_E*
 * code; sg_last_error() returns the thread-local message of the last
 * failure.  Codes map onto the reference's exception taxonomy (errors.py).
 * The library owns all device memory behind handles; the caller owns host
 * buffers.  Calls are not re-entrant per handle.  No torch types anywhere.
 */
#ifndef SIMTGRAPH_CUDA_H
#define SIMTGRAPH_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes -> errors.py classes */
#define SG_OK 0
#define SG_ECONFIG (-1)     /* ConfigError   (errors.py:16-17)  */
#define SG_ERANGE (-2)      /* RangeError    (errors.py:12-13)  */
#define SG_ECONVERGE (-3)   /* ConvergenceError (errors.py:36-45) */
#define SG_ECUDA (-4)       /* SimtGraphError: CUDA failure      */
#define SG_ENOMEM (-5)      /* SimtGraphError: device allocation */
#define SG_EPARSE (-6)      /* ParseError    (errors.py:8-13): malformed input file */
#define SG_EIO (-7)         /* OSError: file cannot be opened / read */

/* apps (apps.py:24; opcodes _kernels_py.py:26-29) */
#define SG_APP_BFS 0
#define SG_APP_SSSP 1
#define SG_APP_CC 2
#define SG_APP_PR 3
#define SG_APP_KCORE 4

/* scheduler kinds (schedulers.py:30) */
#define SG_SCHED_ALB 0
#define SG_SCHED_TWC 1
#define SG_SCHED_LB 2     /* prefix over every active vertex + LB kernel (schedulers.py:280-283) */
#define SG_SCHED_VERTEX 3 /* one thread per active vertex (_kernels_py.py:88-97) */
#define SG_SCHED_EDGE 4   /* contiguous per-thread active-edge ranges (_kernels_py.py:100-117) */

typedef struct sg_graph sg_graph; /* opaque: HBM-resident CSR (+ lazy CSC / sym) */

typedef struct sg_params {
  int32_t app;        /* SG_APP_* */
  int32_t sched;      /* SG_SCHED_* (twc = no huge bin) */
  int32_t blocked;    /* huge-vertex distribution: 0 cyclic, 1 blocked (schedulers.py:191-200) */
  int32_t devices;    /* edge-cut partitions (engine.py:64-85); >1 = simulated on this GPU */
  int64_t source;     /* bfs / sssp (apps.py:83-95) */
  int64_t k;          /* kcore (apps.py:204-208) */
  double damping;     /* pr (apps.py:145-153) */
  double tol;         /* pr */
  int64_t threshold;  /* resolved huge threshold >= 1 (schedulers.py:58-60, worklist.py:122-128) */
  int64_t max_rounds; /* <= 0: 10*V + 256 (engine.py:199-202) */
  int32_t flags;      /* SG_FLAG_* */
  int32_t reserved;
} sg_params;

#define SG_FLAG_TIMING 1  /* fill *ms_out with the CUDA-event time of the BSP loop */
#define SG_FLAG_PROFILE 2 /* host-driven rounds with CUDA events around every kernel
                             (per-kernel times via sg_run_profiled); default is one
                             CUDA-graph launch whose WHILE node runs all rounds */
#define SG_FLAG_TWC_CLASSIC 4 /* TWC CTA bin = one vertex per CTA (the reference's
                                 twc_kernel mapping, _kernels_py.py:140-146) instead of
                                 edge-balanced batches; for the TWC-only ablation */
#define SG_FLAG_RELABEL 8     /* run on the hot-vertex relabeled store (sg_graph.cuh
                                 Relabel): the highest-degree vertices take the low ids
                                 so their labels share L1 lines; labels are mapped back */
#define SG_FLAG_NO_RELABEL 16 /* never relabel.  Neither flag: relabel when devices == 1,
                                 the graph has >= 2^20 vertices and it has been run
                                 before (the build is amortised over repeated runs) */

typedef struct sg_round { /* one BSP round (engine.py:116-163) */
  int64_t frontier_size;  /* RoundRecord.frontier_size */
  int64_t active_edges;   /* RoundRecord.active_edges(): operator applications */
  int64_t huge_count;     /* |huge| after inspection (schedulers.py:291) */
  int64_t huge_edges;     /* PrefixWork.total_edges (lb kernel edges) */
  int64_t large_count;    /* CTA-bin vertices */
  int64_t large_edges;    /* edges of CTA-bin vertices */
  int64_t updated;        /* vertices whose label changed (next frontier / dying) */
  int64_t comm_sent;      /* engine.py:225-229 (devices > 1) */
  int64_t comm_broadcast; /* engine.py:232-234 (devices > 1) */
  int64_t launches_twc;   /* inspect+twc launches: devices with a non-empty local frontier */
  int64_t launches_lb;    /* lb launches: devices whose local frontier had huge vertices */
} sg_round;

const char *sg_last_error(void);
int sg_device_count(int *count);
/* the CUDA device this thread's later calls use (one process per GPU: LOCAL_RANK) */
int sg_set_device(int32_t device);

/* Memory.  Device buffers come from a caching allocator (no cudaMalloc /
 * cudaFree per graph or run after warm-up); sg_release_cached returns the
 * cached blocks to the driver.  sg_host_alloc hands out cached pinned host
 * blocks, e.g. for labels_out (full-speed D2H); release with sg_host_free. */
int sg_host_alloc(int64_t bytes, void **out);
void sg_host_free(void *p);
void sg_release_cached(void);

/* --- graph store (graph.py:29-177) ------------------------------------- */
/* Upload a CSR (graph.py:33-37 dtypes): offsets int64[nv+1], targets int32[ne],
 * weights int64[ne] or NULL.  Validates like Graph._validate (graph.py:44-57).
 * Weights that all fit 1 (2) bytes cross the host link packed (host threads,
 * while the topology is in flight) and are widened back on the device; the
 * graph keeps int64 weights either way.  Pinned host buffers (sg_host_alloc)
 * give full link speed. */
int sg_graph_create(const int64_t *offsets, const int32_t *targets, const int64_t *weights,
                    int64_t nv, int64_t ne, sg_graph **out);
/* generate_rmat on the device (graph.py:274-298), bit-exact to numpy PCG64:
 * pcg = {state_hi, state_lo, inc_hi, inc_lo} of np.random.PCG64(seed).state,
 * cuts = np.cumsum(probs)[:3]. */
int sg_graph_create_rmat(int32_t scale, int64_t edge_factor, const uint64_t pcg[4],
                         const double cuts[3], sg_graph **out);
/* attach_random_weights (graph.py:301-305) on the device for power-of-two
 * ranges (high-low+1 = 2^j <= 2^32): numpy's Lemire path never rejects there. */
int sg_graph_attach_random_weights(sg_graph *g, const uint64_t pcg[4], int64_t low, int64_t high,
                                   sg_graph **out);
/* Upload host weights for an existing device graph (same topology). */
int sg_graph_with_weights(sg_graph *g, const int64_t *weights, sg_graph **out);
/* Graph.load_binary (graph.py:159-177) of an SGB1 file, streamed from disk
 * into HBM through pinned staging blocks (multi-threaded reads overlapped
 * with the H2D copies); Graph._validate (graph.py:44-57) on the device.
 * Bad magic / version: SG_EPARSE; short sections: the reference's
 * ConfigError / RangeError of the arrays numpy would have produced. */
int sg_graph_load_sgb1(const char *path, sg_graph **out);
int sg_graph_info(sg_graph *g, int64_t *nv, int64_t *ne, int32_t *weighted);
/* Copy arrays back to host; any pointer may be NULL.  which: 0 CSR, 1 CSC, 2 symmetrized CSR */
int sg_graph_download(sg_graph *g, int32_t which, int64_t *offsets, int32_t *targets,
                      int64_t *weights);
int sg_graph_view_size(sg_graph *g, int32_t which, int64_t *ne);
/* The derived layouts a graph caches in HBM (like Graph.csc() / symmetrized(),
 * graph.py:102, 117): CSC, symmetrized CSR, pr source blocks, the hot-vertex
 * relabeled store (at most one at a time) and the exact-order pr layouts.
 * sg_graph_release_views drops them all (rebuilt on demand);
 * sg_graph_build_ms reports the last build time of each, in ms:
 * {csc, symmetrized, relabeled store, exact pr layout}. */
int sg_graph_release_views(sg_graph *g);
int sg_graph_build_ms(sg_graph *g, double out[4]);
void sg_graph_destroy(sg_graph *g);

/* --- run level: engine.run (engine.py:190-246) -------------------------- */
int sg_run(sg_graph *g, const sg_params *p, double *labels_out, sg_round *rounds_out,
           int64_t rounds_cap, int64_t *nrounds, double *ms_out);

/* sg_run with hardware load counters: cta_out[r * cta_g + c] = edges processed
 * by the CTAs that ran on SM c (cta_g = SM count) in round r, for the first
 * min(rounds, cta_rounds_cap, 4096) rounds -- the device analogue of the
 * reference's modeled per_cta_edges (simt.py RoundMetrics).  devices == 1. */
int sg_run_cta_counts(sg_graph *g, const sg_params *p, double *labels_out, sg_round *rounds_out,
                      int64_t rounds_cap, int64_t *nrounds, double *ms_out, uint64_t *cta_out,
                      int64_t cta_rounds_cap, int32_t *cta_g);

typedef struct sg_kernel_time { /* per-kernel totals of a profiled run */
  char name[32];
  int64_t launches;
  double ms; /* sum of CUDA-event durations */
} sg_kernel_time;

int sg_run_profiled(sg_graph *g, const sg_params *p, double *labels_out, sg_round *rounds_out,
                    int64_t rounds_cap, int64_t *nrounds, double *ms_out, sg_kernel_time *kt,
                    int32_t kt_cap, int32_t *nkt);

/* --- multi-GPU edge cut (engine.py:64-113): one partition per rank over NCCL.
 * sg_nccl_unique_id on rank 0, broadcast the 128 bytes out of band (e.g.
 * torch.distributed), then every rank calls sg_dist_run on the same graph.
 * All apps: push apps exchange labels by all-reduce(min); pr broadcasts each
 * rank's aux / rank rows; kcore all-reduces alive flags (min) and neighbour
 * marks (max).  labels_out receives the merged labels on every rank. */
int sg_nccl_unique_id(uint8_t id_out[128]);
/* sg_dist_run keeps one NCCL communicator per (id, rank, world) across calls
 * (a unique id bootstraps one communicator); sg_nccl_release destroys them. */
void sg_nccl_release(void);
int sg_dist_run(sg_graph *g, const sg_params *p, const uint8_t nccl_id[128], int32_t rank,
                int32_t world, double *labels_out, sg_round *rounds_out, int64_t rounds_cap,
                int64_t *nrounds, double *ms_out);
/* The same per-rank code path with `world` ranks as host threads sharing this
 * GPU (collectives = device kernels over the ranks' buffers): the multi-rank
 * protocol on one device.  Outputs are rank 0's. */
int sg_dist_run_threads(sg_graph *g, const sg_params *p, int32_t world, double *labels_out,
                        sg_round *rounds_out, int64_t rounds_cap, int64_t *nrounds,
                        double *ms_out);

/* --- multi-GPU edge cut over NVLink peer memory (the B200 transport) ------
 * Replaces the reference's per-device loop + sync_labels (engine.py:64-113,
 * 205-235) with one process per GPU, no collective library in the loop.
 *
 * sg_graph_partition: rows [cuts[rank], cuts[rank+1]) of one view of g (the
 * reference's make_partition cuts, engine.py:64-75) as a graph of their own:
 * kind 0 = CSR rows (+ weights; bfs / sssp), 1 = CSC rows (pr; the full CSR
 * offsets are kept for the out-degrees), 2 = symmetrized rows (cc / kcore).
 * Only the block's edges are stored, so g can be destroyed afterwards.
 * sg_graph_part_info: kind / rank / world, cuts_out[world + 1], edges of the
 * full view.  A partition is run only through sg_team_run.
 * kind may carry SG_PART_RELABEL / SG_PART_NO_RELABEL: the block-local
 * hot-vertex relabeling (every block renumbered onto itself by descending
 * degree, rows sorted -- the kernel layout of the single-device relabeled
 * store, under the reference's cuts; labels come back in the original
 * numbering).  Neither: relabel skewed graphs of >= 2^20 vertices.
 *
 * sg_team_create allocates this rank's symmetric region for nv vertices and
 * exports it (handle_out: 64-byte CUDA IPC handle); after exchanging the
 * handles out of band (e.g. torch.distributed all_gather), sg_team_connect
 * maps every peer's region (handles: world x 64 bytes in rank order).
 * sg_team_run: one BSP run of this rank's partition, the whole loop one
 * CUDA-graph launch; the round's kernels store label updates straight into
 * the owners' / mirrors' regions and synchronise with a device-side barrier
 * (60 s timeout -> SG_ECUDA, the team is then unusable).  p->devices must be
 * the team size.  labels_out gets the merged labels on every rank, rounds_out
 * the global round log (comm_sent / comm_broadcast as engine.py:105-109,
 * 232-234). */
#define SG_PART_RELABEL 0x100
#define SG_PART_NO_RELABEL 0x200
int sg_graph_partition(sg_graph *g, int32_t kind, int32_t world, int32_t rank, sg_graph **out);
int sg_graph_part_info(sg_graph *g, int32_t *kind, int32_t *rank, int32_t *world,
                       int64_t *cuts_out, int64_t *full_ne);
typedef struct sg_team sg_team;
int sg_team_create(int32_t rank, int32_t world, int64_t nv, sg_team **out,
                   uint8_t handle_out[64]);
int sg_team_connect(sg_team *t, const uint8_t *handles);
int sg_team_run(sg_team *t, sg_graph *part, const sg_params *p, double *labels_out,
                sg_round *rounds_out, int64_t rounds_cap, int64_t *nrounds, double *ms_out);
void sg_team_destroy(sg_team *t);
/* The peer transport with `world` ranks as host threads on this GPU (each
 * with its own partition of g and region; peers are plain device pointers).
 * Outputs are rank 0's. */
int sg_peer_run_threads(sg_graph *g, const sg_params *p, int32_t world, double *labels_out,
                        sg_round *rounds_out, int64_t rounds_cap, int64_t *nrounds,
                        double *ms_out);

/* --- kernel level: the reference plugin API (_kernels_py.py:88-201) ------ */
int sg_lb_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                 const double *weights, int64_t nw, const int64_t *huge,
                 const int64_t *cumulative, int64_t nhuge, const double *values, double *out,
                 const double *aux, int64_t naux, int32_t opcode, int32_t blocked,
                 int32_t num_ctas, int32_t threads_per_cta, int32_t warp_size,
                 int64_t *per_cta_edges, int64_t *per_warp_paths, int64_t *accesses);
int sg_twc_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                  const double *weights, int64_t nw, const int64_t *small, int64_t nsmall,
                  const int64_t *medium, int64_t nmedium, const int64_t *large, int64_t nlarge,
                  const double *values, double *out, const double *aux, int64_t naux,
                  int32_t opcode, int32_t num_ctas, int32_t threads_per_cta, int32_t warp_size,
                  int64_t *per_cta_edges);
int sg_vertex_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                     const double *weights, int64_t nw, const int64_t *frontier, int64_t nf,
                     const double *values, double *out, const double *aux, int64_t naux,
                     int32_t opcode, int32_t num_ctas, int32_t threads_per_cta,
                     int64_t *per_cta_edges);
int sg_edge_kernel(const int64_t *offsets, int64_t nv, const int32_t *targets, int64_t ne,
                   const double *weights, int64_t nw, const int64_t *frontier, int64_t nf,
                   const double *values, double *out, const double *aux, int64_t naux,
                   int32_t opcode, int32_t num_ctas, int32_t threads_per_cta,
                   int64_t *per_cta_edges);

/* number of kernels this library launched since load (evidence counter) */
int64_t sg_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif
