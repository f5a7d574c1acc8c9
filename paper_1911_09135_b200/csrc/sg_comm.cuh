// sg_comm.cuh — the label-exchange communicator of the edge-cut BSP
// (sync_labels, engine.py:88-113) behind one interface:
//   * NcclComm   — one process per GPU, NCCL over NVLink / NVSwitch (torchrun);
//   * ThreadComm — `world` host threads sharing ONE GPU (each thread = one
//     rank with its own stream and buffers); the collectives are device
//     kernels over all ranks' buffers.  It runs the exact multi-rank code
//     path on a single B200 (parity tests at world 2..8).
// libnccl is dlopen'ed (the copy torch already loaded when present), so the
// single-GPU library has no NCCL link dependency.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <mutex>

#include "sg_runtime.cuh"

namespace sg {

enum class CType { U8, U32, U64, I64, F64 };
enum class COp { Min, Max, Sum };

inline size_t ctype_size(CType t) {
  switch (t) {
    case CType::U8: return 1;
    case CType::U32: return 4;
    default: return 8;
  }
}

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // in place on `buf` (device memory), ordered on stream s
  virtual void allreduce(void *buf, size_t n, CType t, COp op, cudaStream_t s) = 0;
  virtual void bcast(void *buf, size_t n, CType t, int root, cudaStream_t s) = 0;
  virtual void group_begin() {}
  virtual void group_end() {}
  // personalised exchange: element counts / displacements per peer (host arrays)
  virtual void alltoallv(const void *send, const size_t *scount, const size_t *sdispl, void *recv,
                         const size_t *rcount, const size_t *rdispl, CType t, cudaStream_t s) = 0;
};

// ----------------------------------------------------------------- NCCL --
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};
inline const NcclApi &nccl() {
  static NcclApi n = [] {
    NcclApi x;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
    x.getUniqueId = (decltype(x.getUniqueId))dlsym(h, "ncclGetUniqueId");
    x.commInitRank = (decltype(x.commInitRank))dlsym(h, "ncclCommInitRank");
    x.allReduce = (decltype(x.allReduce))dlsym(h, "ncclAllReduce");
    x.broadcast = (decltype(x.broadcast))dlsym(h, "ncclBroadcast");
    x.send = (decltype(x.send))dlsym(h, "ncclSend");
    x.recv = (decltype(x.recv))dlsym(h, "ncclRecv");
    x.groupStart = (decltype(x.groupStart))dlsym(h, "ncclGroupStart");
    x.groupEnd = (decltype(x.groupEnd))dlsym(h, "ncclGroupEnd");
    x.commDestroy = (decltype(x.commDestroy))dlsym(h, "ncclCommDestroy");
    x.errorString = (decltype(x.errorString))dlsym(h, "ncclGetErrorString");
    return x;
  }();
  if (!n.allReduce || !n.broadcast) throw Error(SG_ECUDA, "libnccl.so.2 not loadable");
  return n;
}
#define SG_NCCL(call)                                                                     \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      throw ::sg::Error(SG_ECUDA, std::string("NCCL: ") + ::sg::nccl().errorString(r_));  \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(const uint8_t id_bytes[128], int rank_, int world_) {
    rank = rank_, world = world_;
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    SG_NCCL(nccl().commInitRank(&comm, world, id, rank));
  }
  ~NcclComm() override {
    if (comm) nccl().commDestroy(comm);
  }
  static ncclDataType_t dt(CType t) {
    switch (t) {
      case CType::U8: return ncclUint8;
      case CType::U32: return ncclUint32;
      case CType::U64: return ncclUint64;
      case CType::I64: return ncclInt64;
      default: return ncclFloat64;
    }
  }
  static ncclRedOp_t rop(COp o) { return o == COp::Min ? ncclMin : o == COp::Max ? ncclMax : ncclSum; }
  void allreduce(void *buf, size_t n, CType t, COp op, cudaStream_t s) override {
    SG_NCCL(nccl().allReduce(buf, buf, n, dt(t), rop(op), comm, s));
  }
  void bcast(void *buf, size_t n, CType t, int root, cudaStream_t s) override {
    SG_NCCL(nccl().broadcast(buf, buf, n, dt(t), root, comm, s));
  }
  void group_begin() override { SG_NCCL(nccl().groupStart()); }
  void group_end() override { SG_NCCL(nccl().groupEnd()); }
  void alltoallv(const void *send, const size_t *scount, const size_t *sdispl, void *recv,
                 const size_t *rcount, const size_t *rdispl, CType t, cudaStream_t s) override {
    const size_t es = ctype_size(t);
    SG_NCCL(nccl().groupStart());
    for (int q = 0; q < world; ++q) {
      if (scount[q])
        SG_NCCL(nccl().send((const char *)send + sdispl[q] * es, scount[q], dt(t), q, comm, s));
      if (rcount[q])
        SG_NCCL(nccl().recv((char *)recv + rdispl[q] * es, rcount[q], dt(t), q, comm, s));
    }
    SG_NCCL(nccl().groupEnd());
  }
};

// ---------------------------------------------------- threads on one GPU --
constexpr int kMaxRanks = 32;
struct RankPtrs {
  void *p[kMaxRanks];
};
template <class T>
__device__ __forceinline__ T cop_apply(COp op, T a, T b) {
  return op == COp::Min ? (b < a ? b : a) : op == COp::Max ? (b > a ? b : a) : a + b;
}
template <class T>
__global__ void k_thread_allreduce(RankPtrs r, int world, size_t n, COp op) {
  const size_t st = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    T x = ((const T *)r.p[0])[i];
    for (int d = 1; d < world; ++d) x = cop_apply(op, x, ((const T *)r.p[d])[i]);
    for (int d = 0; d < world; ++d) ((T *)r.p[d])[i] = x;
  }
}

struct ThreadHub {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  RankPtrs ptrs{};
  const size_t *scount[kMaxRanks], *sdispl[kMaxRanks];
  bool failed = false;
  explicit ThreadHub(int w) : world(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || failed; });
    }
    if (failed) throw Error(SG_ECUDA, "a peer rank failed");
  }
  void fail() {
    std::lock_guard<std::mutex> lk(mu);
    failed = true;
    cv.notify_all();
  }
};

struct ThreadComm : Comm {
  ThreadHub &hub;
  ThreadComm(ThreadHub &h, int rank_) : hub(h) { rank = rank_, world = h.world; }
  void allreduce(void *buf, size_t n, CType t, COp op, cudaStream_t s) override {
    SG_CUDA(cudaStreamSynchronize(s));
    hub.ptrs.p[rank] = buf;
    hub.barrier();
    if (rank == 0 && n) {
      const int g = grid_n((int64_t)n);
      switch (t) {
        case CType::U8: k_thread_allreduce<uint8_t><<<g, 256>>>(hub.ptrs, world, n, op); break;
        case CType::U32: k_thread_allreduce<uint32_t><<<g, 256>>>(hub.ptrs, world, n, op); break;
        case CType::U64:
          k_thread_allreduce<unsigned long long><<<g, 256>>>(hub.ptrs, world, n, op);
          break;
        case CType::I64: k_thread_allreduce<long long><<<g, 256>>>(hub.ptrs, world, n, op); break;
        case CType::F64: k_thread_allreduce<double><<<g, 256>>>(hub.ptrs, world, n, op); break;
      }
      SG_CUDA(cudaGetLastError());
      SG_CUDA(cudaDeviceSynchronize());
    }
    hub.barrier();
  }
  void alltoallv(const void *send, const size_t *scount, const size_t *sdispl, void *recv,
                 const size_t *rcount, const size_t *rdispl, CType t, cudaStream_t s) override {
    SG_CUDA(cudaStreamSynchronize(s));
    hub.ptrs.p[rank] = const_cast<void *>(send);
    hub.scount[rank] = scount, hub.sdispl[rank] = sdispl;
    hub.barrier();
    const size_t es = ctype_size(t);
    for (int q = 0; q < world; ++q) {  // pull what every peer addressed to this rank
      const size_t n = hub.scount[q][rank];
      if (n != rcount[q]) throw Error(SG_ECUDA, "alltoallv: count mismatch");
      if (n)
        SG_CUDA(cudaMemcpyAsync((char *)recv + rdispl[q] * es,
                                (const char *)hub.ptrs.p[q] + hub.sdispl[q][rank] * es, n * es,
                                cudaMemcpyDeviceToDevice, s));
    }
    SG_CUDA(cudaStreamSynchronize(s));
    hub.barrier();
  }
  void bcast(void *buf, size_t n, CType t, int root, cudaStream_t s) override {
    SG_CUDA(cudaStreamSynchronize(s));
    hub.ptrs.p[rank] = buf;
    hub.barrier();
    if (rank == root && n) {
      for (int d = 0; d < world; ++d)
        if (d != root)
          SG_CUDA(cudaMemcpy(hub.ptrs.p[d], buf, n * ctype_size(t), cudaMemcpyDeviceToDevice));
    }
    hub.barrier();
  }
};

// ------------------------------------------------ host-driven dist loops --
struct DistLoop {  // host-driven rounds with a done-flag read back after each
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  DistLoop() {
    SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SG_CUDA(cudaEventCreate(&e0));
    SG_CUDA(cudaEventCreate(&e1));
  }
  ~DistLoop() {
    cudaStreamSynchronize(s);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
  }
  bool done(const Ctl *ctl) {
    Ctl h;
    SG_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    return h.done != 0;
  }
};

inline void dist_results(RunBufs &rb, cudaStream_t s, double *labels_d, int64_t nv, sg_round *rounds_out,
                  int64_t cap, int64_t *nrounds, double *labels_out, int64_t max_rounds) {
  Ctl h;
  SG_CUDA(cudaStreamSynchronize(s));
  SG_CUDA(cudaMemcpy(&h, rb.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
  const int64_t rounds = h.round;
  std::vector<RoundStat> st((size_t)std::min<int64_t>(rounds, rb.stats_cap));
  if (!st.empty())
    SG_CUDA(cudaMemcpy(st.data(), rb.stats.p, sizeof(RoundStat) * st.size(),
                       cudaMemcpyDeviceToHost));
  if (rounds_out && !st.empty())
    std::memcpy(rounds_out, st.data(),
                sizeof(RoundStat) * (size_t)std::min<int64_t>(cap, (int64_t)st.size()));
  *nrounds = rounds;
  if (labels_out)
    SG_CUDA(cudaMemcpy(labels_out, labels_d, sizeof(double) * nv, cudaMemcpyDeviceToHost));
  if (h.error == SG_ECONVERGE)
    throw Error(SG_ECONVERGE, "did not converge within " + std::to_string(max_rounds) + " rounds");
  if (h.error) throw Error(h.error, "round log capacity exhausted");
}


// one rank of the bitmap-frontier push apps (sg_dist_push.cu)
void run_push_dist(Graph &g, const sg_params &p, int64_t thr, int64_t max_rounds, Comm &cm,
                   double *labels_out, sg_round *rounds_out, int64_t cap, int64_t *nrounds,
                   double *ms_out);

}  // namespace sg
