// Ping-pong latency between two CTAs through global memory (profiling aid):
// one-way store->load visibility, with relaxed.gpu / volatile accesses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pp profiles/mb_pingpong.cu && /tmp/pp
#include <cuda_runtime.h>
#include <cstdio>

__global__ void pingpong(unsigned long long* flag, int iters, int far, long long* out) {
  // CTA 0 and CTA `far` (others idle)
  if (blockIdx.x != 0 && blockIdx.x != (unsigned)far) return;
  if (threadIdx.x != 0) return;
  const bool ping = blockIdx.x == 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const unsigned long long want = 2ull * i + (ping ? 0 : 1);
    if (ping) {
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(want + 1) : "memory");
      unsigned long long v;
      do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory"); } while (v != want + 2);
    } else {
      unsigned long long v;
      do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory"); } while (v != want);
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(want + 1) : "memory");
    }
  }
  if (ping) *out = clock64() - t0;
}

int main() {
  unsigned long long* flag;
  long long* out;
  cudaMalloc(&flag, 256);
  cudaMalloc(&out, 8);
  int G;
  cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int far : {1, 2, 37, 74, 100, 147}) {
    cudaMemset(flag, 0, 256);
    const int iters = 2000;
    pingpong<<<G, 32>>>(flag, iters, far, out);
    long long cyc;
    cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("partner CTA %3d: round trip %.0f cycles = %.3f us (clock %d MHz) %s\n", far, (double)cyc / iters,
           (double)cyc / iters / (clk / 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
