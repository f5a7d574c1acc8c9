// Microbenchmarks for an order-exact (sequential) f64 row sum on B200:
//  (1) dependent DADD latency; (2) one thread summing an L2-resident buffer in
//  order, values staged through shared memory by the other warps of its CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

__global__ void k_chain(double* out, double c, long n) {
  double x = out[0];
#pragma unroll 1
  for (long i = 0; i < n; i += 8) {
    x = x + c; x = x + c; x = x + c; x = x + c;
    x = x + c; x = x + c; x = x + c; x = x + c;
  }
  out[1] = x;
}

// CTA of 256 threads: warps 1..7 (and warp 0 lanes) copy tiles of T doubles
// into a ring of smem tiles, thread 0 adds them in order.
template <int T, int NT>
__global__ void k_seq(const double* __restrict__ v, long n, double* out) {
  __shared__ double ring[NT][T];
  __shared__ volatile int ready[NT];
  __shared__ volatile int consumed;
  int tid = threadIdx.x;
  if (tid < NT) ready[tid] = -1;
  if (tid == 0) consumed = -1;
  __syncthreads();
  long ntiles = (n + T - 1) / T;
  if (tid < 32) {
    if (tid == 0) {
      double s = 0.0;
      for (long t = 0; t < ntiles; ++t) {
        int slot = t % NT;
        while (ready[slot] != (int)t) {}
        long m = n - t * T < T ? n - t * T : T;
        const double* r = ring[slot];
        if (m == T) {
#pragma unroll 16
          for (int i = 0; i < T; ++i) s += r[i];
        } else {
          for (int i = 0; i < m; ++i) s += r[i];
        }
        consumed = (int)t;
      }
      out[0] = s;
    }
    return;
  }
  // producers: warps 1..7, each tile copied by all 224 producer threads
  int p = tid - 32, np = blockDim.x - 32;
  for (long t = 0; t < ntiles; ++t) {
    int slot = t % NT;
    if (t >= NT) { while (consumed < (int)(t - NT)) {} }
    long base = t * T;
    for (int i = p; i < T; i += np) if (base + i < n) ring[slot][i] = __ldg(v + base + i);
    asm volatile("bar.sync 1, %0;" ::"r"(np));
    if (p == 0) { __threadfence_block(); ready[slot] = (int)t; }
  }
}

double ref_sum(const std::vector<double>& h) { double s = 0; for (double x : h) s += x; return s; }

int main() {
  double* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  long n = 1 << 24;
  k_chain<<<1, 1>>>(d, 1e-3, n); cudaDeviceSynchronize();
  cudaEventRecord(a); k_chain<<<1, 1>>>(d, 1e-3, n); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"dadd_chain_ns\": %.3f, \"dadd_cycles_at_max\": %.2f}\n", ms * 1e6 / n, ms * 1e-3 / n * clk * 1e3);
  for (long m : {370000L, 560000L, 2000000L}) {
    std::vector<double> h(m);
    unsigned long long st = 12345;
    for (auto& x : h) { st = st * 6364136223846793005ULL + 1442695040888963407ULL; x = (st >> 11) * 0x1.0p-53 * 3.0; }
    double* dv; cudaMalloc(&dv, m * 8); cudaMemcpy(dv, h.data(), m * 8, cudaMemcpyHostToDevice);
    double* o; cudaMalloc(&o, 8);
    k_seq<256, 8><<<1, 256>>>(dv, m, o); cudaDeviceSynchronize();
    cudaEventRecord(a); k_seq<256, 8><<<1, 256>>>(dv, m, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double got; cudaMemcpy(&got, o, 8, cudaMemcpyDeviceToHost);
    printf("{\"n\": %ld, \"seq_ms\": %.4f, \"ns_per_add\": %.3f, \"exact\": %d}\n", m, ms, ms * 1e6 / m, got == ref_sum(h));
    cudaFree(dv); cudaFree(o);
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
