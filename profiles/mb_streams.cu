// Microbenchmark: HBM read bandwidth vs the number of concurrent read
// streams, the access pattern of DIA SpMV (ndiag streams of the diagonal
// data + one written stream).  Each variant sums S arrays of n doubles
// (stride n apart, the DIA data layout) into y.  Prints GB/s per S for a
// plain grid-stride thread-per-row kernel (k_dia's structure without x) and
// for a TMA bulk-copy variant is NOT included — this isolates the stream
// count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_streams mb_streams.cu && ./mb_streams
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) k_sum(long n, int S, const double* __restrict__ d, double* __restrict__ y) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    int k = 0;
    for (; k + U <= S; k += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(d + (long)(k + u) * n + i));
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u];
    }
    for (; k < S; ++k) acc += d[(long)k * n + i];
    y[i] = acc;
  }
}

int main() {
  const long n = 216000000L / 4;   // 54 M rows
  const int SMAX = 27;
  double *d, *y;
  cudaMalloc(&d, (size_t)n * SMAX * 8);
  cudaMalloc(&y, (size_t)n * 8);
  cudaMemset(d, 0, (size_t)n * SMAX * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int S : {1, 2, 4, 8, 12, 16, 20, 27}) {
    for (int variant = 0; variant < 2; ++variant) {
      const int grid = sms * 8;
      for (int w = 0; w < 2; ++w) {
        if (variant == 0) k_sum<4><<<grid, 256>>>(n, S, d, y); else k_sum<8><<<grid, 256>>>(n, S, d, y);
      }
      cudaEventRecord(a);
      const int reps = 10;
      for (int r = 0; r < reps; ++r) {
        if (variant == 0) k_sum<4><<<grid, 256>>>(n, S, d, y); else k_sum<8><<<grid, 256>>>(n, S, d, y);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= reps;
      const double bytes = (double)n * 8 * (S + 1);
      printf("{\"streams\": %d, \"unroll\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", S, variant ? 8 : 4, ms, bytes / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
