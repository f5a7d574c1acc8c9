// Microbenchmark: random 4-byte gather throughput (the label access of every
// push kernel) on B200.  col[] streams (coalesced), lab[col[e]] is random.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int U, int MODE>
__global__ void __launch_bounds__(256) k_gather(const uint32_t *__restrict__ col, const uint32_t *lab, int64_t n,
                                                unsigned long long *out) {
  uint32_t acc = 0;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n; b += st * U) {
    uint32_t d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = (b + u * st < n) ? __ldcs(col + b + u * st) : 0;
    uint32_t x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) x[u] = lab[d[u]];
      else x[u] = __ldcg(lab + d[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += x[u];
  }
  if (acc == 0x12345) atomicAdd(out, 1ull);
}

int main() {
  const int64_t n = 256ll << 20;  // edges
  const int logv = 24;
  std::vector<uint32_t> h(n);
  std::mt19937_64 rng(1);
  for (auto &x : h) x = (uint32_t)(rng() & ((1u << logv) - 1));
  uint32_t *col, *lab;
  unsigned long long *out;
  cudaMalloc(&col, n * 4);
  cudaMalloc(&lab, (1ll << 26) * 4);
  cudaMalloc(&out, 8);
  cudaMemset(lab, 0, (1ll << 26) * 4);
  cudaMemcpy(col, h.data(), n * 4, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char *name, auto kern, int per_sm) {
    for (int it = 0; it < 3; ++it) kern<<<sms * per_sm, 256>>>(col, lab, n, out);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) kern<<<sms * per_sm, 256>>>(col, lab, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-28s blocks/SM %d: %.3f ms  %.1f G gathers/s\n", name, per_sm, ms, n / ms / 1e6);
  };
  for (int per_sm : {4, 8}) {
    run("U4 ld (L1)", k_gather<4, 0>, per_sm);
    run("U4 ld.cg (L2)", k_gather<4, 1>, per_sm);
    run("U8 ld (L1)", k_gather<8, 0>, per_sm);
    run("U8 ld.cg (L2)", k_gather<8, 1>, per_sm);
    run("U16 ld.cg (L2)", k_gather<16, 1>, per_sm);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
