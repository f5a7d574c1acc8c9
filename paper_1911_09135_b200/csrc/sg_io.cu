// sg_io.cu — SGB1 binary graphs straight into HBM (reference graph.py:136-177).
//
// Layout (little-endian, graph.py:138-143):
//   "SGB1" | u32 version (1) | u8 weighted | 3 pad | u64 V | u64 E |
//   int64 offsets[V+1] | int32 targets[E] | int64 weights[E] (if weighted)
//
// The reference parses the file into numpy arrays and then builds the Graph
// (validation, graph.py:44-57).  Here the sections stream from the file into
// a ring of pinned staging blocks (several reader threads per block) while
// the copy engine moves the previous block to its place in the device CSR;
// the reference's validation then runs as one device pass, reporting the
// first failing check in the reference's order with its message.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sg_graph.cuh"

namespace sg {
namespace {

constexpr size_t kStage = 64ull << 20;  // bytes per pinned staging block
constexpr int kRing = 3;                // staging blocks in flight

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// pread exactly n bytes at off (several threads for large blocks)
void read_block(int fd, char *dst, size_t n, int64_t off) {
  const int T = (int)std::max<size_t>(1, std::min<size_t>(8, n >> 22));  // >= 4 MB per thread
  auto part = [&](int t, std::string *err) {
    const size_t a = n * t / T, b = n * (t + 1) / T;
    size_t done = a;
    while (done < b) {
      const ssize_t r = pread(fd, dst + done, b - done, off + (int64_t)done);
      if (r <= 0) {
        *err = r == 0 ? "unexpected end of file" : std::string("read failed: ") + strerror(errno);
        return;
      }
      done += (size_t)r;
    }
  };
  std::vector<std::string> errs((size_t)T);
  if (T == 1) {
    part(0, &errs[0]);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(part, t, &errs[(size_t)t]);
    for (auto &x : th) x.join();
  }
  for (auto &e : errs)
    if (!e.empty()) throw Error(SG_EPARSE, e);
}

// file section [off, off + n) -> device dst, double-buffered through pinned blocks
struct Streamer {
  int fd;
  cudaStream_t s;
  char *buf[kRing];
  cudaEvent_t ev[kRing];
  int next = 0;
  void copy(void *dst, int64_t off, size_t n) {
    for (size_t done = 0; done < n;) {
      const size_t c = std::min(kStage, n - done);
      const int b = next;
      next = (next + 1) % kRing;
      SG_CUDA(cudaEventSynchronize(ev[b]));  // block b's previous copy has drained
      read_block(fd, buf[b], c, off + (int64_t)done);
      SG_CUDA(cudaMemcpyAsync((char *)dst + done, buf[b], c, cudaMemcpyHostToDevice, s));
      SG_CUDA(cudaEventRecord(ev[b], s));
      done += c;
    }
  }
};

// graph.py:44-57 checks that need the arrays: bit 0 offsets decrease, bit 1
// a target outside [0, V)
__global__ void k_validate(const int64_t *__restrict__ off, int64_t nv,
                           const uint32_t *__restrict__ col, int64_t ne,
                           unsigned int *__restrict__ flags) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool dec = false, out = false;
  for (int64_t v = t0; v < nv; v += st) dec |= off[v + 1] < off[v];
  for (int64_t i = t0; i < ne; i += st) out |= (int64_t)(int32_t)col[i] < 0 || (int64_t)col[i] >= nv;
  const unsigned m = (dec ? 1u : 0u) | (out ? 2u : 0u);
  const unsigned w = __reduce_or_sync(0xffffffffu, m);
  if ((threadIdx.x & 31u) == 0 && w) atomicOr(flags, w);
}

}  // namespace
}  // namespace sg

extern "C" int sg_graph_load_sgb1(const char *path, sg_graph **out) {
  using sg::Error;
  return sg::guard([&] {
    if (!path || !out) throw Error(SG_ECONFIG, "null argument");
    sg::Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) throw Error(SG_EIO, std::string("cannot open ") + path + ": " + strerror(errno));
    struct stat stt;
    if (fstat(f.fd, &stt) != 0) throw Error(SG_EIO, std::string("stat failed: ") + strerror(errno));
    const int64_t fsize = (int64_t)stt.st_size;
    unsigned char h[32] = {0};
    const ssize_t hr = pread(f.fd, h, sizeof(h), 0);
    if (hr < 4 || std::memcmp(h, "SGB1", 4) != 0)
      throw Error(SG_EPARSE, "bad magic; not a simtgraph binary graph");
    uint32_t version = 0;
    std::memcpy(&version, h + 4, 4);
    if (hr < 8 || version != 1)
      throw Error(SG_EPARSE, "unsupported binary version " + std::to_string(version));
    const bool weighted = h[8] != 0;
    uint64_t nv_u = 0, ne_u = 0;
    if (hr >= 20) std::memcpy(&nv_u, h + 12, 8);
    if (hr >= 28) std::memcpy(&ne_u, h + 20, 8);
    // what numpy's frombuffer would have produced from a short file: the
    // sections as far as the file goes (graph.py:168-174), then Graph's checks
    const int64_t body = std::max<int64_t>(0, fsize - 28);
    const int64_t nv_hdr = (int64_t)nv_u, ne_hdr = (int64_t)ne_u;
    if (nv_u > (1ull << 40) || ne_u > (1ull << 40))
      throw Error(SG_ECONFIG, "offsets must have num_vertices+1 entries starting at 0");
    const int64_t n_off = std::min<int64_t>(nv_hdr + 1, body / 8);
    const int64_t rest = body - n_off * 8;
    const int64_t ne = std::min<int64_t>(ne_hdr, std::max<int64_t>(0, rest) / 4);  // len(targets)
    const int64_t rest2 = rest - ne * 4;
    const int64_t n_w = weighted ? std::min<int64_t>(ne_hdr, std::max<int64_t>(0, rest2) / 8) : 0;
    // Graph() takes num_vertices = len(offsets) - 1 (graph.py:38)
    if (n_off < 1) throw Error(SG_ECONFIG, "offsets must have num_vertices+1 entries starting at 0");
    const int64_t nv = n_off - 1;
    if (nv > 0x7fffffffLL) throw Error(SG_ERANGE, "vertex ids must fit int32");

    auto g = std::make_shared<sg::Graph>();
    g->nv = nv, g->ne = ne;
    g->csr.nv = nv, g->csr.ne = ne;
    g->csr.off.alloc(nv + 1);
    g->csr.col.alloc(ne ? ne : 1);
    if (weighted) g->w64.alloc(n_w ? n_w : 1);
    cudaStream_t s;
    SG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    sg::Streamer st{f.fd, s, {}, {}, 0};
    for (int b = 0; b < sg::kRing; ++b) {
      st.buf[b] = (char *)sg::host_alloc(sg::kStage);
      cudaEventCreateWithFlags(&st.ev[b], cudaEventDisableTiming);
    }
    auto cleanup = [&] {
      cudaStreamSynchronize(s);
      for (int b = 0; b < sg::kRing; ++b) {
        sg::host_free(st.buf[b]);
        cudaEventDestroy(st.ev[b]);
      }
      cudaStreamDestroy(s);
    };
    try {
      int64_t pos = 28;  // header: magic 4 + u32 4 + u8 + 3 pad + u64 V + u64 E
      st.copy(g->csr.off.p, pos, sizeof(int64_t) * (size_t)(nv + 1));
      pos += 8 * (nv + 1);
      if (ne) st.copy(g->csr.col.p, pos, sizeof(int32_t) * (size_t)ne);
      pos += 4 * ne;
      if (n_w) st.copy(g->w64.p, pos, sizeof(int64_t) * (size_t)n_w);
      SG_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    // Graph._validate (graph.py:44-57), in its order
    int64_t ends[2] = {0, 0};
    SG_CUDA(cudaMemcpy(&ends[0], g->csr.off.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
    SG_CUDA(cudaMemcpy(&ends[1], g->csr.off.p + nv, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (ends[0] != 0) throw Error(SG_ECONFIG, "offsets must have num_vertices+1 entries starting at 0");
    if (ends[1] != ne) throw Error(SG_ECONFIG, "offsets must end at num_edges");
    sg::DBuf<unsigned int> flags(1);
    SG_CUDA(cudaMemset(flags.p, 0, sizeof(unsigned int)));
    const int grid = sg::sm_info().sms * 8;
    SG_LAUNCH(sg::k_validate, grid, 256, 0, 0, g->csr.off.p, nv, g->csr.col.p, ne, flags.p);
    unsigned int fl = 0;
    SG_CUDA(cudaMemcpy(&fl, flags.p, sizeof(fl), cudaMemcpyDeviceToHost));
    if (fl & 1u) throw Error(SG_ECONFIG, "offsets must be non-decreasing");
    if (fl & 2u) throw Error(SG_ERANGE, "edge target outside 0..num_vertices-1");
    if (weighted && n_w != ne) throw Error(SG_ECONFIG, "weights must align with targets");
    if (weighted) sg::weights_finalize(*g);
    *out = new sg_graph{g};
  });
}
