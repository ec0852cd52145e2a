// Microbenchmark for the SM-resident MGS kernel design (profiling aid, not
// shipped).  Variants isolate the grid barrier, the shared-memory w slice and
// the L2 prefetch.  Build+run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb profiles/mb_mgs.cu && /tmp/mb
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int PB = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <bool SYNC>
__device__ __forceinline__ double red(double v, double* gparts, unsigned* counter, int pass, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < (PB / 32) ? scratch[lane] : 0.0;
    t = warp_sum(t);
    const int slot = pass & 1;
    if (SYNC) {
      if (lane == 0) {
        gparts[slot * gridDim.x + blockIdx.x] = t;
        __threadfence();
        atomicAdd(counter, 1u);
        const unsigned target = (unsigned)(pass + 1) * gridDim.x;
        unsigned seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
        } while (seen < target);
      }
      __syncwarp();
      __threadfence();
      double g = 0.0;
      for (unsigned b = lane; b < gridDim.x; b += 32) g += __ldcg(gparts + slot * gridDim.x + b);
      t = warp_sum(g);
    }
    if (lane == 0) scratch[32 + slot] = t;
  }
  __syncthreads();
  return scratch[32 + (pass & 1)] * 1e-30;
}

// tag barrier: (value, tag) slots, readers poll the tags directly
struct alignas(16) Part {
  double v;
  unsigned long long tag;
};
__device__ __forceinline__ double red_tag(double v, Part* parts, unsigned long long tag, int pass, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < (PB / 32) ? scratch[lane] : 0.0;
    t = warp_sum(t);
    Part* slots = parts + (pass & 1) * gridDim.x;
    if (lane == 0) {
      slots[blockIdx.x].v = t;
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&slots[blockIdx.x].tag), "l"(tag) : "memory");
    }
    double g = 0.0;
    for (unsigned b = lane; b < gridDim.x; b += 32) {
      unsigned long long seen;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(&slots[b].tag) : "memory");
      } while (seen != tag);
      g += __ldcg(&slots[b].v);
    }
    g = warp_sum(g);
    if (lane == 0) scratch[32 + (pass & 1)] = g;
  }
  __syncthreads();
  return scratch[32 + (pass & 1)] * 1e-30;
}

template <int U>
__global__ void __launch_bounds__(PB, 1) ktag(double* V, int64_t n, int64_t ld, int j, int64_t chunk, Part* parts,
                                            unsigned long long epoch, double* out) {
  extern __shared__ double ws[];
  double* scratch = ws + chunk;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = n < lo + chunk ? n : lo + chunk;
  const int len = hi > lo ? (int)(hi - lo) : 0;
  double h = 0.5;
  for (int i = 1; i <= j; ++i) {
    const double* vp = V + (int64_t)(i - 1) * ld + lo;
    const double* vi = V + (int64_t)i * ld + lo;
    double acc = 0.0;
    for (int k0 = threadIdx.x; k0 < len; k0 += U * PB) {
      double a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k0 + u * PB;
        a[u] = kk < len ? __ldcs(vp + kk) : 0.0;
        b[u] = kk < len ? __ldcg(vi + kk) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k0 + u * PB;
        if (kk < len) {
          const double w = ws[kk] - h * a[u];
          ws[kk] = w;
          acc += b[u] * w;
        }
      }
    }
    h = 0.5 + red_tag(acc, parts, (epoch << 8) | (unsigned long long)i, i, scratch);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = h;
}

float run_tag(double* V, int64_t n, int64_t ld, int j, Part* parts, double* out) {
  static unsigned long long epoch = 1;
  int G = 148;
  int64_t chunk = (((n + G - 1) / G) + 1) & ~int64_t(1);
  size_t smem = chunk * 8 + 34 * 8;
  cudaFuncSetAttribute(ktag<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 6; ++rep) {
    ++epoch;
    void* args[] = {&V, &n, &ld, &j, &chunk, &parts, &epoch, &out};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((const void*)ktag<8>, dim3(G), dim3(PB), args, smem, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  printf("%-28s j=%d  %8.1f us  per pass %6.2f us  %s\n", "tag barrier (smem,U8)", j, best * 1e3, best * 1e3 / j,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  return best;
}

template <bool SYNC, bool SMEM, bool PREF, int U>
__global__ void __launch_bounds__(PB, 1) k(double* V, int64_t n, int64_t ld, int j, int64_t chunk, double* gparts,
                                         unsigned* counter, double* out) {
  extern __shared__ double ws[];
  double* scratch = ws + (SMEM ? chunk : 0);
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = n < lo + chunk ? n : lo + chunk;
  const int len = hi > lo ? (int)(hi - lo) : 0;
  double h = 0.5;
  double reg = 0.0;
  for (int i = 1; i <= j; ++i) {
    const double* vp = V + (int64_t)(i - 1) * ld + lo;
    const double* vi = V + (int64_t)i * ld + lo;
    if (PREF && i + 1 <= j) {
      const char* base = reinterpret_cast<const char*>(V + (int64_t)(i + 1) * ld + lo);
      const int64_t bytes = ((int64_t)len * 8) & ~int64_t(15);
      for (int64_t off = (int64_t)threadIdx.x * 16384; off < bytes; off += 16384LL * PB) {
        const uint32_t sz = (uint32_t)(bytes - off < 16384 ? bytes - off : 16384);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(sz) : "memory");
      }
    }
    double acc = 0.0;
    for (int k0 = threadIdx.x; k0 < len; k0 += U * PB) {
      double a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k0 + u * PB;
        a[u] = kk < len ? __ldcs(vp + kk) : 0.0;
        b[u] = kk < len ? __ldcg(vi + kk) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k0 + u * PB;
        if (kk < len) {
          if (SMEM) {
            const double w = ws[kk] - h * a[u];
            ws[kk] = w;
            acc += b[u] * w;
          } else {
            reg = reg - h * a[u];
            acc += b[u] * reg;
          }
        }
      }
    }
    h = 0.5 + red<SYNC>(acc, gparts, counter, i - 1, scratch);   // barrier index from 0
  }
  if (threadIdx.x == 0) out[blockIdx.x] = h + reg;
}

template <bool SYNC, bool SMEM, bool PREF, int U>
float run(const char* name, double* V, int64_t n, int64_t ld, int j, double* gp, unsigned* ctr, double* out) {
  int G = 148;
  int64_t chunk = (((n + G - 1) / G) + 1) & ~int64_t(1);
  size_t smem = (SMEM ? chunk : 0) * 8 + 34 * 8;
  cudaFuncSetAttribute(k<SYNC, SMEM, PREF, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 6; ++rep) {
    cudaMemset(ctr, 0, 4);
    void* args[] = {&V, &n, &ld, &j, &chunk, &gp, &ctr, &out};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((const void*)k<SYNC, SMEM, PREF, U>, dim3(G), dim3(PB), args, smem, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  printf("%-28s j=%d  %8.1f us  per pass %6.2f us  %s\n", name, j, best * 1e3, best * 1e3 / j,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  return best;
}

int main() {
  const int64_t n = 4000000, ld = (n + 31) & ~31LL;
  const int m = 30;
  double* V;
  cudaMalloc(&V, (m + 1) * ld * 8);
  cudaMemset(V, 0, (m + 1) * ld * 8);
  double *gp, *out;
  unsigned* ctr;
  cudaMalloc(&gp, 4096);
  cudaMalloc(&ctr, 64);
  cudaMalloc(&out, 4096);
  // pure barrier cost: tiny vectors, so the pass body is negligible
  run<true, true, false, 8>("barrier only (n=296)", V, 296, 320, 20, gp, ctr, out);
  run<false, true, false, 8>("no barrier (n=296)", V, 296, 320, 20, gp, ctr, out);
  Part* parts;
  cudaMalloc(&parts, 2 * 148 * sizeof(Part));
  cudaMemset(parts, 0, 2 * 148 * sizeof(Part));
  for (int j : {1, 20}) {
    run_tag(V, n, ld, j, parts, out);
    run<true, true, true, 8>("full (sync,smem,pref,U8)", V, n, ld, j, gp, ctr, out);
    run<true, true, false, 8>("no prefetch", V, n, ld, j, gp, ctr, out);
    run<true, true, true, 4>("U4", V, n, ld, j, gp, ctr, out);
    run<false, true, true, 8>("no grid sync", V, n, ld, j, gp, ctr, out);
    run<true, false, true, 8>("no smem w", V, n, ld, j, gp, ctr, out);
    run<false, false, false, 8>("loads only", V, n, ld, j, gp, ctr, out);
  }
  return 0;
}
