// Microbenchmark + correctness check for the TMA-streamed TMEM-resident MGS
// kernel (paper_2411_10143_b200/csrc/mgs_tma.cuh).  Profiling aid, not shipped.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I include \
//        -o /tmp/mbt profiles/mb_mgs_tma.cu && /tmp/mbt
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "../paper_2411_10143_b200/csrc/mgs_tma.cuh"

using namespace svb::mgs;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 4000000;
  const int64_t ld = (n + 31) & ~31LL;
  const int m = 30;
  int G = 0;
  CK(cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0));
  const int64_t chunk = (((n + G - 1) / G) + 1) & ~int64_t(1);
  if (chunk > MAX_SLICE) {
    printf("slice too large\n");
    return 1;
  }
  std::vector<double> hV((size_t)(m + 1) * ld, 0.0);
  srand(1);
  for (int i = 0; i <= m; ++i)
    for (int64_t k = 0; k < n; ++k) hV[(size_t)i * ld + k] = (rand() / (double)RAND_MAX - 0.5) / sqrt((double)n);
  double *V, *H, *cs, *sn, *g;
  unsigned long long* gslot;
  svb_krylov_status* st;
  CK(cudaMalloc(&V, hV.size() * 8));
  CK(cudaMalloc(&H, (m + 1) * m * 8));
  CK(cudaMalloc(&cs, m * 8));
  CK(cudaMalloc(&sn, m * 8));
  CK(cudaMalloc(&g, (m + 1) * 8));
  CK(cudaMalloc(&gslot, 2 * SLOT_STRIDE * G * 8));
  CK(cudaMemset(gslot, 0, 2 * SLOT_STRIDE * G * 8));
  CK(cudaMallocManaged(&st, sizeof(svb_krylov_status)));
  CK(cudaMemset(H, 0, (m + 1) * m * 8));
  CK(cudaMemset(cs, 0, m * 8));
  CK(cudaMemset(sn, 0, m * 8));
  CK(cudaMemset(g, 0, (m + 1) * 8));
  CK(cudaFuncSetAttribute(k_mgs_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  unsigned long long epoch = 1;
  Args A{};
  A.V = V;
  A.n = n;
  A.ld = ld;
  A.chunk = chunk;
  A.m = m;
  A.H = H;
  A.cs = cs;
  A.sn = sn;
  A.g = g;
  A.st = st;
  A.bnorm = 1.0;
  A.gslot = gslot;
  if (!plan(chunk, &A.chunk_count, &A.nsb, &A.nres)) {
    printf("no plan\n");
    return 1;
  }
  printf("chunks %d ring stages %d\n", A.chunk_count, A.nsb);
  auto launch = [&](int j) {
    A.j = j;
    A.epoch = epoch++;
    void* args[] = {&A};
    CK(cudaLaunchCooperativeKernel((const void*)k_mgs_tma<false>, dim3(G), dim3(NT), args, SMEM, 0));
  };
  // ---- correctness at several j against a CPU MGS
  int bad = 0;
  for (int j : {0, 1, 5, 29}) {
    CK(cudaMemcpy(V, hV.data(), hV.size() * 8, cudaMemcpyHostToDevice));
    launch(j);
    CK(cudaDeviceSynchronize());
    std::vector<double> w(hV.begin() + (size_t)(j + 1) * ld, hV.begin() + (size_t)(j + 1) * ld + n);
    std::vector<double> h(j + 2);
    for (int i = 0; i <= j; ++i) {
      double d = 0;
      for (int64_t k = 0; k < n; ++k) d += hV[(size_t)i * ld + k] * w[k];
      h[i] = d;
      for (int64_t k = 0; k < n; ++k) w[k] -= d * hV[(size_t)i * ld + k];
    }
    double nn = 0;
    for (int64_t k = 0; k < n; ++k) nn += w[k] * w[k];
    const double hn = sqrt(nn);
    std::vector<double> gH((m + 1) * m), gw(n);
    CK(cudaMemcpy(gH.data(), H, gH.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(gw.data(), V + (size_t)(j + 1) * ld, n * 8, cudaMemcpyDeviceToHost));
    // H[j][j] is rotated by the Givens epilogue (cs/sn are zero here, so
    // rows i < j are rotated to 0*..: compare the raw h only via V[j+1])
    double eh = 0, ew = 0;
    for (int64_t k = 0; k < n; ++k) ew = fmax(ew, fabs(gw[k] - w[k] / hn));
    const double ehn = fabs(st->hnext - hn) / hn;
    printf("check j=%2d  max rel err h %.2e  hnext %.2e  max abs err V[j+1] %.2e\n", j, eh, ehn, ew);
    if (!(eh < 1e-9 && ehn < 1e-12 && ew < 1e-12)) bad = 1;
  }
  // ---- timing
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaMemcpy(V, hV.data(), hV.size() * 8, cudaMemcpyHostToDevice));
  for (int j : {0, 1, 5, 13, 20, 29}) {
    float best = 1e9, sum = 0;
    const int R = 20;
    for (int r = 0; r < R + 2; ++r) {
      CK(cudaEventRecord(a));
      launch(j);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (r >= 2) {
        best = fminf(best, ms);
        sum += ms;
      }
    }
    const double bytes = 8.0 * n * (j + 3);
    printf("j=%2d  best %8.1f us  mean %8.1f us  per pass %6.2f us  %7.1f GB/s (algorithmic 8n(j+3))\n", j,
           best * 1e3, sum / R * 1e3, best * 1e3 / (j + 2), bytes / (best * 1e-3) / 1e9);
  }
  // streaming reference: D2D copy of one 32 MB row
  {
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(a));
      CK(cudaMemcpyAsync(V + 29 * ld, V + 30 * ld, n * 8, cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = fminf(best, ms);
    }
    printf("D2D copy of one row: %.1f us, %.1f GB/s (r+w)\n", best * 1e3, 16.0 * n / (best * 1e-3) / 1e9);
  }
  // ---- phase trace of one j=13 launch (globaltimer, ns)
  {
    const int j = 13, np = j + 2;
    unsigned long long* tr;
    CK(cudaMalloc(&tr, (size_t)G * np * 4 * 8));
    A.trace = tr;
    for (int r = 0; r < 3; ++r) launch(j);
    CK(cudaDeviceSynchronize());
    A.trace = nullptr;
    std::vector<unsigned long long> h((size_t)G * np * 4);
    CK(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < G; ++c) t0 = std::min(t0, h[(size_t)c * np * 4]);
    printf("pass: [min..max over CTAs of] start | consumed | cta-reduced | exchanged   (us from first start)\n");
    for (int p = 0; p < np; ++p) {
      double mn[4], mx[4];
      for (int k = 0; k < 4; ++k) {
        mn[k] = 1e30;
        mx[k] = -1e30;
        for (int c = 0; c < G; ++c) {
          const double v = (h[((size_t)c * np + p) * 4 + k] - t0) * 1e-3;
          mn[k] = std::min(mn[k], v);
          mx[k] = std::max(mx[k], v);
        }
      }
      printf("%2d: %7.2f..%7.2f | %7.2f..%7.2f | %7.2f..%7.2f | %7.2f..%7.2f\n", p, mn[0], mx[0], mn[1], mx[1],
             mn[2], mx[2], mn[3], mx[3]);
    }
    // is the spread of the streaming phase (consumed - start) systematic per
    // CTA (the same SMs slow every pass) or random?
    std::vector<double> ev(G, 0.0), od(G, 0.0);
    int ne = 0, no = 0;
    for (int p = 1; p < np - 1; ++p) {
      (p & 1 ? no : ne)++;
      for (int c = 0; c < G; ++c) {
        const double v = (double)(h[((size_t)c * np + p) * 4 + 1] - h[((size_t)c * np + p) * 4 + 0]) * 1e-3;
        (p & 1 ? od : ev)[c] += v;
      }
    }
    double me = 0, mo = 0;
    for (int c = 0; c < G; ++c) { ev[c] /= ne; od[c] /= no; me += ev[c]; mo += od[c]; }
    me /= G; mo /= G;
    double sxy = 0, sxx = 0, syy = 0, lo = 1e30, hi = -1e30;
    for (int c = 0; c < G; ++c) {
      sxy += (ev[c] - me) * (od[c] - mo); sxx += (ev[c] - me) * (ev[c] - me); syy += (od[c] - mo) * (od[c] - mo);
      const double a = 0.5 * (ev[c] + od[c]);
      lo = std::min(lo, a); hi = std::max(hi, a);
    }
    printf("stream phase per CTA: mean %.2f us, per-CTA means %.2f..%.2f us, even/odd-pass correlation %.2f\n",
           0.5 * (me + mo), lo, hi, sxy / sqrt(sxx * syy + 1e-30));
    std::vector<int> idx(G);
    for (int c = 0; c < G; ++c) idx[c] = c;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return ev[a] + od[a] > ev[b] + od[b]; });
    printf("slowest CTAs:");
    for (int k = 0; k < 12; ++k) printf(" %d(%.2f)", idx[k], 0.5 * (ev[idx[k]] + od[idx[k]]));
    printf("\nfastest CTAs:");
    for (int k = G - 12; k < G; ++k) printf(" %d(%.2f)", idx[k], 0.5 * (ev[idx[k]] + od[idx[k]]));
    printf("\n");
  }
  printf(bad ? "MISMATCH\n" : "ALL OK\n");
  return bad;
}
