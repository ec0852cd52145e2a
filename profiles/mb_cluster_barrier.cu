// Grid all-reduce through thread-block clusters (profiling aid): partials
// folded inside each cluster over distributed shared memory, cluster leaders
// exchange through tagged global slots, result broadcast back over DSMEM.
// Compared with the flat all-CTA tagged exchange of the Arnoldi kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cb profiles/mb_cluster_barrier.cu && /tmp/cb
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;
constexpr int NT = 288;
constexpr int PASSES = 64;
constexpr int STRIDE = 32;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// tagged exchange among `n` participants (index `me`), warp-collective
__device__ double tag_exchange(unsigned long long* sl, int n, int me, double part, unsigned want) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(part);
    const unsigned long long w0 = ((unsigned long long)want << 32) | (bits >> 32),
                             w1 = ((unsigned long long)want << 32) | (bits & 0xffffffffull);
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(sl + STRIDE * me), "l"(w0), "l"(w1) : "memory");
  }
  double v[8];
  unsigned pending = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[k] = 0.0;
    if (lane + 32 * k < n) pending |= 1u << k;
  }
  while (__any_sync(0xffffffffu, pending != 0)) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (pending & (1u << k)) {
        unsigned long long w0, w1;
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(sl + STRIDE * (lane + 32 * k)) : "memory");
        if ((w0 >> 32) == want && (w1 >> 32) == want) {
          v[k] = __longlong_as_double((long long)((w0 << 32) | (w1 & 0xffffffffull)));
          pending &= ~(1u << k);
        }
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  return wsum(s);
}

template <bool CLUSTER>
__global__ void kbar(unsigned long long* slots, unsigned epoch, double* out) {
  __shared__ double part[2], total[2];
  const int warp = threadIdx.x >> 5;
  double h = 1.0;
  cg::cluster_group cl = cg::this_cluster();
  const int C = CLUSTER ? (int)cl.num_blocks() : 1;
  const int crank = CLUSTER ? (int)cl.block_rank() : 0;
  const int nleaders = gridDim.x / C;
  const int me = blockIdx.x / C;
  for (int p = 0; p < PASSES; ++p) {
    const int b = p & 1;
    const unsigned want = (epoch << 8) | (unsigned)(p + 1);
    unsigned long long* sl = slots + (size_t)b * STRIDE * 256;
    const double mine = h * 1e-3 + blockIdx.x;
    if (!CLUSTER) {
      __syncthreads();
      if (warp == 0) {
        const double t = tag_exchange(sl, gridDim.x, blockIdx.x, mine, want);
        if ((threadIdx.x & 31) == 0) total[b] = t;
      }
      __syncthreads();
      h = total[b];
      continue;
    }
    if (threadIdx.x == 0) part[b] = mine;
    cl.sync();
    if (crank == 0 && warp == 0) {
      double s = 0.0;
      for (int r = 0; r < C; ++r) s += *cl.map_shared_rank(&part[b], r);   // fixed order
      const double t = tag_exchange(sl, nleaders, me, s, want);
      if ((threadIdx.x & 31) == 0) total[b] = t;
    }
    cl.sync();
    h = *cl.map_shared_rank(&total[b], 0);
  }
  if (CLUSTER) cl.sync();   // no CTA may exit while a peer still reads its shared memory
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = h;
}

template <bool CLUSTER>
void run(const char* name, int C, unsigned long long* slots, double* out) {
  static unsigned epoch = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = 0;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (!CLUSTER) {   // cooperative launch does not combine with clusters: all 148
    at[na].id = cudaLaunchAttributeCooperative;   // CTAs fit at once anyway
    at[na].val.cooperative = 1;
    ++na;
  }
  if (CLUSTER) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = C;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    int maxc = 0;
    cudaLaunchConfig_t q = cfg;
    q.attrs = at;
    q.numAttrs = 1;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&maxc, (const void*)kbar<CLUSTER>, &q);
    if (oe != cudaSuccess) printf("  occupancy query: %s\n", cudaGetErrorString(oe));
    printf("  cluster %d: max active clusters %d (need %d)\n", C, maxc, 148 / C);
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    unsigned e = epoch++;
    cudaEventRecord(a);
    void* args[] = {&slots, &e, &out};
    cudaError_t err = cudaLaunchKernelExC(&cfg, (const void*)kbar<CLUSTER>, args);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (err != cudaSuccess) {
      printf("%-32s launch failed: %s\n", name, cudaGetErrorString(err));
      return;
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2 && ms < best) best = ms;
  }
  printf("%-32s %7.3f us per exchange %s\n", name, best * 1e3 / PASSES, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* slots;
  double* out;
  cudaMalloc(&slots, 2 * STRIDE * 256 * 8);
  cudaMemset(slots, 0, 2 * STRIDE * 256 * 8);
  cudaMalloc(&out, 8);
  run<false>("flat, 148 CTAs", 1, slots, out);
  run<true>("cluster 2 (74 leaders)", 2, slots, out);
  run<true>("cluster 4 (37 leaders)", 4, slots, out);
  return 0;
}
