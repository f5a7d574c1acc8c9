// Cost of the system-scope primitives the peer barrier is built from, one
// thread, averaged over many iterations inside one kernel (B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence fence.cu && ./fence
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long flag[64];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <int MODE>
__global__ void k(int iters, unsigned long long *out, unsigned long long *remote) {
  if (threadIdx.x) return;
  unsigned long long *f = remote ? remote : flag;
  const unsigned long long t0 = gt();
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) acc += i;
    if (MODE == 1) __threadfence_system();
    if (MODE == 2) __threadfence();
    if (MODE == 3) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"((unsigned long long)i) : "memory");
    if (MODE == 4) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      acc += v;
    }
    if (MODE == 5) {  // release store + acquire poll of the same word (world-1 barrier)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"((unsigned long long)i + 1) : "memory");
      unsigned long long v;
      do asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      while (v < (unsigned long long)i + 1);
    }
    if (MODE == 6) {
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f), "l"((unsigned long long)i + 1) : "memory");
      unsigned long long v;
      do asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      while (v < (unsigned long long)i + 1);
    }
    if (MODE == 7) {  // relaxed sys store + poll, fence.acq_rel.sys around
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f), "l"((unsigned long long)i + 1) : "memory");
      unsigned long long v;
      do asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      while (v < (unsigned long long)i + 1);
      asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
  }
  out[0] = gt() - t0;
  out[1] = acc;
}
int main() {
  unsigned long long *d;
  cudaMalloc(&d, 16);
  const char *names[] = {"loop", "fence.sc.sys", "fence.sc.gpu", "st.release.sys", "ld.acquire.sys",
                         "st.release.sys+ld.acquire.sys poll", "st.release.gpu+ld.acquire.gpu poll",
                         "fence.acq_rel.sys+relaxed st/poll+fence"};
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 8; ++m) {
      switch (m) {
        case 0: k<0><<<1, 32>>>(iters, d, nullptr); break;
        case 1: k<1><<<1, 32>>>(iters, d, nullptr); break;
        case 2: k<2><<<1, 32>>>(iters, d, nullptr); break;
        case 3: k<3><<<1, 32>>>(iters, d, nullptr); break;
        case 4: k<4><<<1, 32>>>(iters, d, nullptr); break;
        case 5: k<5><<<1, 32>>>(iters, d, nullptr); break;
        case 6: k<6><<<1, 32>>>(iters, d, nullptr); break;
        case 7: k<7><<<1, 32>>>(iters, d, nullptr); break;
      }
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      if (rep) printf("%-45s %8.1f ns\n", names[m], (double)h[0] / iters);
    }
  // empty-kernel launch + the barrier-kernel shape, host-timed with events
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int m : {0, 5}) {
    cudaEventRecord(e0);
    for (int i = 0; i < 1000; ++i) {
      if (m == 0) k<0><<<1, 32>>>(1, d, nullptr);
      else k<5><<<1, 32>>>(1, d, nullptr);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("back-to-back launches, mode %d: %.2f us each\n", m, ms);
  }
  return 0;
}
