// Device-resident Krylov building blocks: restarted MGS-GMRES (solver.py:
// 219-342) and Hestenes-Stiefel CG (new).
//
// Every reduction is a single kernel: CTAs reduce a fixed grid-stride share
// of the vectors, write a per-CTA partial, and the last CTA to finish
// (atomic ticket) folds the partials in a fixed tree order and runs the
// scalar epilogue (Givens rotation, CG alpha/beta, convergence estimate).
// Results are therefore deterministic run to run, scalars never leave the
// device inside an iteration, and the host reads one mapped status block
// per iteration.  The modified Gram-Schmidt loop is fused as
// "axpy_{i-1} + dot_i" passes: pass i reads w, V[i-1] and V[i] once.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "matrix.cuh"
#include "mgs_tma.cuh"

struct svb_krylov {
  int64_t n = 0, ld = 0;
  int m = 0;
  unsigned rgrid = 1;
  svb::Buf V, x, b, tmp, p, q, r;
  svb::Buf H, cs, sn, g, y, scal, partials, counter;
  svb_krylov_status* st_host = nullptr;
  svb_krylov_status* st_dev = nullptr;
  // SM-resident MGS (k_gm_mgs_resident): rows per CTA, dynamic smem bytes,
  // per-CTA partial slots; `normalized` = column whose V[j+1] the fused
  // kernel already normalised
  int64_t chunk = 0;
  size_t res_smem = 0;
  bool resident = false;
  bool tmem = false;        // use the TMEM-staged variant (k_gm_mgs_tmem)
  size_t tmem_smem = 0;
  int normalized = -1;
  svb::Buf gparts;
  // TMA-streamed MGS (mgs_tma.cuh, the default when the slice fits): launch
  // plan, tagged exchange slots and the per-launch epoch of the tags
  bool tma = false;
  int tma_chunks = 0, tma_stages = 0, tma_nres = 0;
  int tma_grid = 0;          // CTAs of the TMA Arnoldi kernel (mgs_grid)
  int64_t tma_chunk = 0;     // its slice length
  unsigned long long epoch = 0;
  svb::Buf gslot;
  // recorded right after every status-producing kernel: the host waits on
  // this, not on the stream, so work enqueued behind it (the speculative
  // next SpMV, CG's p update) overlaps the host's decision
  cudaEvent_t ev = nullptr;
  svb::Buf ctl, hist;   // batched-CG control block and estimate log
  unsigned dgrid = 1;
  svb::Buf dparts;      // fused DIA SpMV+dot partials (dgrid doubles + counter)
  int64_t hist_cap = 0;
  ~svb_krylov() {
    if (ev) cudaEventDestroy(ev);
    if (st_host) cudaFreeHost(st_host);
  }
};

struct svb_vecops {
  int64_t n = 0;
  unsigned grid = 1;
  svb::Buf partials;  // grid doubles + reduction counter
  svb::Buf bpart;     // block sweeps: grid x (VB+1) doubles + counter (lazy)
  svb::Buf spart;     // fused SpMV+dot: sgrid doubles + counter (lazy)
  unsigned sgrid = 0;
};

namespace svb {

constexpr int KB = 256;  // threads per CTA for the Krylov kernels
// longest restart: y (m doubles) must fit k_gm_update_x's dynamic shared
// memory next to its 8.3 KB static triangle
constexpr int KRYLOV_MAX_M = 24000;
enum { S_RR = 0, S_ALPHA = 1, S_BETA = 2 };

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// grid-stride over element pairs (rows are 256-byte aligned), odd tail on
// thread 0 of CTA 0
template <class F2, class F1>
__device__ __forceinline__ void for_pairs(int64_t n, F2 f2, F1 f1) {
  const int64_t n2 = n >> 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x)
    f2(2 * i);
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) f1(n - 1);
}

// Block-sum `v`, publish the CTA partial, and return true in the last CTA
// (all threads), where `*total` (thread 0) is the fixed-order grand total.
__device__ bool grid_sum_last(double v, double* partials, unsigned* counter, double* total) {
  __shared__ double sh[KB / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < KB / 32; ++w) b += sh[w];
    partials[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double t = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += KB) t += __ldcg(partials + i);
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  if (lane == 0) sh[wid] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int w = 0; w < KB / 32; ++w) g += sh[w];
    *total = g;
    *counter = 0;  // ready for the next reduction on this stream
  }
  return true;
}

__device__ __forceinline__ bool bad(double v) { return !isfinite(v); }

// ---------------------------------------------------------------------------
// GMRES
// ---------------------------------------------------------------------------
struct Gm {
  double* V;
  int64_t n, ld;
  int m;
  double *H, *cs, *sn, *g, *y;
  double* partials;
  unsigned* counter;
  svb_krylov_status* st;
};

// ||b|| or ||b - tmp|| into st->beta
__global__ void __launch_bounds__(KB) k_resnorm(const double* __restrict__ b, const double* __restrict__ t,
                                                int64_t n, double* partials, unsigned* counter,
                                                svb_krylov_status* st) {
  double acc = 0.0;
  for_pairs(
      n,
      [&](int64_t e) {
        double2 bb = ld2(b + e);
        double2 tt = t ? ld2(t + e) : make_double2(0.0, 0.0);
        double r0 = bb.x - tt.x, r1 = bb.y - tt.y;
        acc += r0 * r0;
        acc += r1 * r1;
      },
      [&](int64_t e) {
        double r0 = b[e] - (t ? t[e] : 0.0);
        acc += r0 * r0;
      });
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) {
    st->beta = sqrt(tot);
    st->nonfinite = bad(st->beta);
  }
}

// r = b - tmp into V0 and ||r||; the next kernel scales V0 by 1/beta
__global__ void __launch_bounds__(KB) k_gm_residual(Gm G, const double* __restrict__ b,
                                                    const double* __restrict__ t) {
  double acc = 0.0;
  double* v0 = G.V;
  for_pairs(
      G.n,
      [&](int64_t e) {
        double2 bb = ld2(b + e), tt = ld2(t + e);
        double2 r = make_double2(bb.x - tt.x, bb.y - tt.y);
        st2(v0 + e, r);
        acc += r.x * r.x;
        acc += r.y * r.y;
      },
      [&](int64_t e) {
        double r = b[e] - t[e];
        v0[e] = r;
        acc += r * r;
      });
  double tot;
  if (grid_sum_last(acc, G.partials, G.counter, &tot) && threadIdx.x == 0) {
    const double beta = sqrt(tot);
    G.st->beta = beta;
    G.st->nonfinite = bad(beta);
    G.g[0] = beta;   // H, cs, sn and g[1..m] were cleared by the host's memsets
  }
}

// V[j] /= d where d = g[0] (restart) or the recorded hnext
__global__ void __launch_bounds__(KB) k_gm_scale(double* __restrict__ v, int64_t n,
                                                 const double* __restrict__ dptr) {
  const double d = *dptr;
  for_pairs(
      n,
      [&](int64_t e) {
        double2 a = ld2(v + e);
        st2(v + e, make_double2(a.x / d, a.y / d));
      },
      [&](int64_t e) { v[e] = v[e] / d; });
}

// pass 0: H[0,j] = V0 . w   (w = V[j+1])
__global__ void __launch_bounds__(KB) k_gm_dot0(Gm G, int j) {
  const double* __restrict__ w = G.V + (int64_t)(j + 1) * G.ld;
  const double* __restrict__ v = G.V;
  double acc = 0.0;
  for_pairs(
      G.n,
      [&](int64_t e) {
        double2 a = ld2(v + e), c = ld2(w + e);
        acc += a.x * c.x;
        acc += a.y * c.y;
      },
      [&](int64_t e) { acc += v[e] * w[e]; });
  double tot;
  if (grid_sum_last(acc, G.partials, G.counter, &tot) && threadIdx.x == 0) G.H[j] = tot;
}

// pass i (1..j): w -= H[i-1,j] V[i-1];  H[i,j] = V[i] . w
__global__ void __launch_bounds__(KB) k_gm_pass(Gm G, int i, int j) {
  double* __restrict__ w = G.V + (int64_t)(j + 1) * G.ld;
  const double* __restrict__ vp = G.V + (int64_t)(i - 1) * G.ld;
  const double* __restrict__ vi = G.V + (int64_t)i * G.ld;
  const double h = G.H[(i - 1) * G.m + j];
  double acc = 0.0;
  for_pairs(
      G.n,
      [&](int64_t e) {
        double2 ww = ld2(w + e), a = ld2(vp + e), c = ld2(vi + e);
        ww.x -= h * a.x;
        ww.y -= h * a.y;
        st2(w + e, ww);
        acc += c.x * ww.x;
        acc += c.y * ww.y;
      },
      [&](int64_t e) {
        double ww = w[e] - h * vp[e];
        w[e] = ww;
        acc += vi[e] * ww;
      });
  double tot;
  if (grid_sum_last(acc, G.partials, G.counter, &tot) && threadIdx.x == 0) G.H[i * G.m + j] = tot;
}

// final pass: w -= H[j,j] V[j]; hnext = ||w||; Givens update of column j,
// residual estimate |g[j+1]|/||b|| (solver.py:294-313)
__global__ void __launch_bounds__(KB) k_gm_final(Gm G, int j, double bnorm) {
  double* __restrict__ w = G.V + (int64_t)(j + 1) * G.ld;
  const double* __restrict__ vj = G.V + (int64_t)j * G.ld;
  const double h = G.H[j * G.m + j];
  double acc = 0.0;
  for_pairs(
      G.n,
      [&](int64_t e) {
        double2 ww = ld2(w + e), a = ld2(vj + e);
        ww.x -= h * a.x;
        ww.y -= h * a.y;
        st2(w + e, ww);
        acc += ww.x * ww.x;
        acc += ww.y * ww.y;
      },
      [&](int64_t e) {
        double ww = w[e] - h * vj[e];
        w[e] = ww;
        acc += ww * ww;
      });
  double tot;
  if (grid_sum_last(acc, G.partials, G.counter, &tot) && threadIdx.x == 0) {
    const int m = G.m;
    double* H = G.H;
    const double hnext = sqrt(tot);
    for (int i = 0; i < j; ++i) {
      const double a = H[i * m + j], b = H[(i + 1) * m + j];
      const double hi = G.cs[i] * a + G.sn[i] * b;
      H[(i + 1) * m + j] = -G.sn[i] * a + G.cs[i] * b;
      H[i * m + j] = hi;
    }
    const double hjj = H[j * m + j];
    const double denom = hypot(hjj, hnext);
    double c = 1.0, s = 0.0;
    if (denom != 0.0) {
      c = hjj / denom;
      s = hnext / denom;
    }
    G.cs[j] = c;
    G.sn[j] = s;
    H[j * m + j] = c * hjj + s * hnext;
    G.g[j + 1] = -s * G.g[j];
    G.g[j] = c * G.g[j];
    H[(j + 1) * m + j] = hnext;  // kept for V[j+1] /= hnext
    const double est = fabs(G.g[j + 1]) / bnorm;
    G.st->hnext = hnext;
    G.st->hjj = H[j * m + j];
    G.st->estimate = est;
    G.st->nonfinite = bad(hnext) || bad(est);
  }
}

// ---------------------------------------------------------------------------
// SM-resident MGS: one persistent cooperative kernel per Arnoldi step.
// CTA c (one per SM) owns rows [c*chunk, (c+1)*chunk) and keeps its slice of
// w in shared memory for the whole orthogonalisation, so every pass streams
// only the basis rows: w never round-trips through L2/HBM.  Passes are
// separated by grid barriers; each CTA folds the per-CTA partials of a dot
// product in the same fixed order, so every CTA holds the identical h_i
// without a second barrier.  The final pass also normalises V[j+1] and CTA 0
// runs the Givens epilogue.
// ---------------------------------------------------------------------------
constexpr int PB = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order CTA sum, result returned to every thread
__device__ __forceinline__ double cta_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < (PB / 32) ? scratch[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) scratch[32] = t;
  }
  __syncthreads();
  const double r = scratch[32];
  __syncthreads();
  return r;
}

// grid-wide fixed-order sum of one partial per CTA (double-buffered slots)
__device__ __forceinline__ double grid_sum(double part, double* gparts, int slot, double* scratch,
                                           cooperative_groups::grid_group& grid) {
  if (threadIdx.x == 0) gparts[slot * gridDim.x + blockIdx.x] = part;
  grid.sync();
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) t += __ldcg(gparts + slot * gridDim.x + b);
    t = warp_sum(t);
    if (threadIdx.x == 0) scratch[33] = t;
  }
  __syncthreads();
  const double r = scratch[33];
  __syncthreads();
  return r;
}

// Lean CTA+grid reduction for the resident MGS kernel: two block barriers
// per pass.  Warp partials go to shared memory; warp 0 folds them, publishes
// the CTA partial, arrives on a monotonic grid counter (zeroed by the host
// before the launch) and spins until all CTAs of this pass arrived, then
// folds the per-CTA partials in fixed order.  Every CTA computes the same
// total, so no broadcast barrier is needed.
__device__ __forceinline__ double fused_grid_sum(double v, double* gparts, unsigned* counter, int pass,
                                                 double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < (PB / 32) ? scratch[lane] : 0.0;
    t = warp_sum(t);
    const int slot = pass & 1;
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
    g = warp_sum(g);
    if (lane == 0) scratch[32 + slot] = g;
  }
  __syncthreads();
  return scratch[32 + (pass & 1)];
}

__device__ void givens_epilogue(Gm& G, int j, double hnext, double bnorm) {
  const int m = G.m;
  double* H = G.H;
  for (int i = 0; i < j; ++i) {
    const double a = H[i * m + j], b = H[(i + 1) * m + j];
    const double hi = G.cs[i] * a + G.sn[i] * b;
    H[(i + 1) * m + j] = -G.sn[i] * a + G.cs[i] * b;
    H[i * m + j] = hi;
  }
  const double hjj = H[j * m + j];
  const double denom = hypot(hjj, hnext);
  double c = 1.0, s = 0.0;
  if (denom != 0.0) {
    c = hjj / denom;
    s = hnext / denom;
  }
  G.cs[j] = c;
  G.sn[j] = s;
  H[j * m + j] = c * hjj + s * hnext;
  G.g[j + 1] = -s * G.g[j];
  G.g[j] = c * G.g[j];
  H[(j + 1) * m + j] = hnext;
  const double est = fabs(G.g[j + 1]) / bnorm;
  G.st->hnext = hnext;
  G.st->hjj = H[j * m + j];
  G.st->estimate = est;
  G.st->nonfinite = bad(hnext) || bad(est);
}

// Bulk L2 prefetch (TMA engine, cp.async.bulk.prefetch.L2) of this CTA's
// slice of the basis row the NEXT pass reads: the DRAM stream for pass i+1
// overlaps pass i's arithmetic and grid barrier, so pass loads hit L2.
__device__ __forceinline__ void prefetch_slice_l2(const double* p, int len) {
  const char* base = reinterpret_cast<const char*>(p);
  const int64_t bytes = ((int64_t)len * 8) & ~int64_t(15);
  constexpr int64_t PIECE = 16384;
  for (int64_t off = (int64_t)threadIdx.x * PIECE; off < bytes; off += PIECE * PB) {
    const uint32_t sz = (uint32_t)(bytes - off < PIECE ? bytes - off : PIECE);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(sz) : "memory");
  }
}

__global__ void __launch_bounds__(PB, 1) k_gm_mgs_resident(Gm G, int j, double bnorm, int64_t chunk,
                                                          double* gparts, unsigned* gcounter) {
  extern __shared__ double ws[];
  double* scratch = ws + chunk;  // 34 doubles
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = G.n < lo + chunk ? G.n : lo + chunk;
  const int len = hi > lo ? (int)(hi - lo) : 0;
  double* wg = G.V + (int64_t)(j + 1) * G.ld + lo;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  auto row = [&](int i) { return G.V + (int64_t)i * G.ld + lo; };

  // Element k of this CTA's slice is handled by thread k % PB; batches of U
  // elements per thread keep 2U independent loads in flight.  The first
  // batch of the NEXT pass is loaded into registers before each grid
  // barrier, so the barrier's latency overlaps those loads; the rest of the
  // next pass's rows are pulled into L2 by a bulk prefetch.  The basis rows
  // are read-only here (V[j+1] is written only after the last read).
  constexpr int U = 8;
  double pa[U], pb[U];   // preloaded first batch of the coming pass
  auto preload = [&](const double* a, const double* b) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = threadIdx.x + u * PB;
      pa[u] = k < len ? __ldcs(a + k) : 0.0;
      pb[u] = (b != nullptr && k < len) ? __ldcg(b + k) : 0.0;
    }
  };

  // pass 0: stage w, h_0 = V_0 . w
  double acc = 0.0;
  if (j >= 1) prefetch_slice_l2(row(1), len);
  {
    const double* v0 = row(0);
    for (int k0 = threadIdx.x; k0 < len; k0 += U * PB) {
      double a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * PB;
        a[u] = k < len ? __ldcs(wg + k) : 0.0;
        b[u] = k < len ? __ldcg(v0 + k) : 0.0;   // reused next pass: keep in L2
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * PB;
        if (k < len) ws[k] = a[u];
        acc += b[u] * a[u];
      }
    }
  }
  preload(row(0), j >= 1 ? row(1) : nullptr);
  double h = fused_grid_sum(acc, gparts, gcounter, 0, scratch);
  if (lead) G.H[j] = h;

  // passes 1..j: w -= h_{i-1} V_{i-1};  h_i = V_i . w
  for (int i = 1; i <= j; ++i) {
    const double* vp = row(i - 1);
    const double* vi = row(i);
    if (i + 1 <= j) prefetch_slice_l2(row(i + 1), len);
    acc = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {   // preloaded first batch
      const int k = threadIdx.x + u * PB;
      if (k < len) {
        const double w = ws[k] - h * pa[u];
        ws[k] = w;
        acc += pb[u] * w;
      }
    }
    for (int k0 = threadIdx.x + U * PB; k0 < len; k0 += U * PB) {
      double a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * PB;
        a[u] = k < len ? __ldcs(vp + k) : 0.0;   // second and last use (L2 hit)
        b[u] = k < len ? __ldcg(vi + k) : 0.0;   // reused next pass: keep in L2
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * PB;
        if (k < len) {
          const double w = ws[k] - h * a[u];
          ws[k] = w;
          acc += b[u] * w;
        }
      }
    }
    preload(vi, i + 1 <= j ? row(i + 1) : nullptr);
    h = fused_grid_sum(acc, gparts, gcounter, i, scratch);
    if (lead) G.H[i * G.m + j] = h;
  }

  // final: w -= h_j V_j; hnext = ||w||; V[j+1] = w / hnext
  acc = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int k = threadIdx.x + u * PB;
    if (k < len) {
      const double w = ws[k] - h * pa[u];
      ws[k] = w;
      acc += w * w;
    }
  }
  {
    const double* vj = row(j);
    for (int k0 = threadIdx.x + U * PB; k0 < len; k0 += U * PB) {
      double a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * PB;
        a[u] = k < len ? __ldcs(vj + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * PB;
        if (k < len) {
          const double w = ws[k] - h * a[u];
          ws[k] = w;
          acc += w * w;
        }
      }
    }
  }
  const double hnext = sqrt(fused_grid_sum(acc, gparts, gcounter, j + 1, scratch));
#pragma unroll 4
  for (int k = threadIdx.x; k < len; k += PB) wg[k] = ws[k] / hnext;
  if (lead) givens_epilogue(G, j, hnext, bnorm);
}

// ---------------------------------------------------------------------------
// TMEM-staged SM-resident MGS (the default on sm_100a when the slice fits).
//
// Same pass structure as k_gm_mgs_resident, but each basis row is read from
// HBM exactly once per Arnoldi step: pass i loads V_i's slice for the dot
// product and parks it in tensor memory (TMEM, 256 KB/SM, otherwise idle in
// this bandwidth-bound kernel); pass i+1 applies w -= h_i V_i from TMEM
// instead of re-reading V_i through L2.  w stays in shared memory.  Traffic
// per step is the algorithmic minimum 8n(j+3) bytes and L2->SM traffic is
// halved.  TMEM layout: a thread owns TMEM lane 32*(warp%4)+lane and the 64
// columns [64*(warp/4), +64), i.e. up to 32 doubles (elements tid+u*PB).
// ---------------------------------------------------------------------------
constexpr int TMEM_COLS = 512;
constexpr int TMEM_MAX_PER_THREAD = 32;  // doubles per thread (64 columns)
constexpr int TB = 8;                    // doubles per tcgen05 batch (.x16)

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const double* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, double* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(PB, 1) k_gm_mgs_tmem(Gm G, int j, double bnorm, int64_t chunk,
                                                      double* gparts, unsigned* gcounter) {
  extern __shared__ double ws[];
  double* scratch = ws + chunk;  // 34 doubles
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // this thread's lane quadrant and column block
  const uint32_t my_tmem = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));

  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = G.n < lo + chunk ? G.n : lo + chunk;
  const int len = hi > lo ? (int)(hi - lo) : 0;
  const int nbatch = (len + TB * PB - 1) / (TB * PB);   // uniform across the CTA
  double* wg = G.V + (int64_t)(j + 1) * G.ld + lo;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  auto row = [&](int i) { return G.V + (int64_t)i * G.ld + lo; };

  // pass 0: stage w in smem, V_0 in TMEM, h_0 = V_0 . w
  double acc = 0.0;
  if (j >= 1) prefetch_slice_l2(row(1), len);
  {
    const double* v0 = row(0);
    for (int bt = 0; bt < nbatch; ++bt) {
      double a[TB], b[TB];
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int k = threadIdx.x + (bt * TB + u) * PB;
        a[u] = k < len ? __ldcs(wg + k) : 0.0;
        b[u] = k < len ? __ldcs(v0 + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int k = threadIdx.x + (bt * TB + u) * PB;
        if (k < len) ws[k] = a[u];
        acc += b[u] * a[u];
      }
      tmem_st16(my_tmem + 16 * bt, b);
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  double h = fused_grid_sum(acc, gparts, gcounter, 0, scratch);
  if (lead) G.H[j] = h;

  // passes 1..j: w -= h_{i-1} V_{i-1} (TMEM);  h_i = V_i . w;  V_i -> TMEM
  for (int i = 1; i <= j; ++i) {
    const double* vi = row(i);
    if (i + 1 <= j) prefetch_slice_l2(row(i + 1), len);
    acc = 0.0;
    for (int bt = 0; bt < nbatch; ++bt) {
      double b[TB], p[TB];
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int k = threadIdx.x + (bt * TB + u) * PB;
        b[u] = k < len ? __ldcs(vi + k) : 0.0;
      }
      tmem_ld16(my_tmem + 16 * bt, p);
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int k = threadIdx.x + (bt * TB + u) * PB;
        if (k < len) {
          const double w = ws[k] - h * p[u];
          ws[k] = w;
          acc += b[u] * w;
        }
      }
      tmem_st16(my_tmem + 16 * bt, b);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    h = fused_grid_sum(acc, gparts, gcounter, i, scratch);
    if (lead) G.H[i * G.m + j] = h;
  }

  // final: w -= h_j V_j (TMEM); hnext = ||w||; V[j+1] = w / hnext
  acc = 0.0;
  for (int bt = 0; bt < nbatch; ++bt) {
    double p[TB];
    tmem_ld16(my_tmem + 16 * bt, p);
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const int k = threadIdx.x + (bt * TB + u) * PB;
      if (k < len) {
        const double w = ws[k] - h * p[u];
        ws[k] = w;
        acc += w * w;
      }
    }
  }
  const double hnext = sqrt(fused_grid_sum(acc, gparts, gcounter, j + 1, scratch));
#pragma unroll 4
  for (int k = threadIdx.x; k < len; k += PB) wg[k] = ws[k] / hnext;
  if (lead) givens_epilogue(G, j, hnext, bnorm);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
}

// Back substitution for y in the reference order (solver.py:211-214) on one
// thread, from H and g in global memory: the restart lengths (j+1 > 32) whose
// triangle does not fit the per-CTA staging of k_gm_update_x.
__global__ void k_gm_solve_y(Gm G, int j) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const int m = G.m;
  for (int i = j; i >= 0; --i) {
    double dot = 0.0;
    for (int k = i + 1; k <= j; ++k) dot += G.H[i * m + k] * G.y[k];
    G.y[i] = (G.g[i] - dot) / G.H[i * m + i];
  }
}

// x += V[:j+1]^T y (solver.py:215-216, 339-340).  For j+1 <= 32 every CTA
// first solves the (j+1)x(j+1) triangular system for y itself (solver.py:
// 211-214, at most ~1K flops, from H in L2), which replaces a separate
// one-thread launch; longer restarts take y from k_gm_solve_y (G.y) into
// dynamic shared memory (ys, j+1 doubles).
__global__ void __launch_bounds__(KB) k_gm_update_x(Gm G, int j, double* __restrict__ x) {
  extern __shared__ double ys[];
  __shared__ double hs[32 * 32 + 32];   // the (j+1)^2 triangle of H and g, staged once
  const int m = G.m, nj = j + 1;
  if (nj <= 32) {
    for (int t = threadIdx.x; t < nj * nj; t += blockDim.x) hs[t] = G.H[(t / nj) * m + (t % nj)];
    for (int t = threadIdx.x; t < nj; t += blockDim.x) hs[nj * nj + t] = G.g[t];
    __syncthreads();
    if (threadIdx.x == 0) {
      // back substitution in the reference order (solver.py:211-214)
      for (int i = j; i >= 0; --i) {
        double dot = 0.0;
        for (int k = i + 1; k <= j; ++k) dot += hs[i * nj + k] * ys[k];
        ys[i] = (hs[nj * nj + i] - dot) / hs[i * nj + i];
      }
      if (blockIdx.x == 0)
        for (int i = 0; i <= j; ++i) G.y[i] = ys[i];
    }
  } else {
    for (int t = threadIdx.x; t < nj; t += blockDim.x) ys[t] = G.y[t];
  }
  __syncthreads();
  for_pairs(
      G.n,
      [&](int64_t e) {
        double2 t = make_double2(0.0, 0.0);
        int i = 0;
        for (; i + 8 <= nj; i += 8) {   // 8 rows' loads in flight, summed in row order
          double2 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = ld2(G.V + (int64_t)(i + u) * G.ld + e);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            t.x += v[u].x * ys[i + u];
            t.y += v[u].y * ys[i + u];
          }
        }
        for (; i <= j; ++i) {
          double2 v = ld2(G.V + (int64_t)i * G.ld + e);
          t.x += v.x * ys[i];
          t.y += v.y * ys[i];
        }
        double2 xx = ld2(x + e);
        st2(x + e, make_double2(xx.x + t.x, xx.y + t.y));
      },
      [&](int64_t e) {
        double t = 0.0;
        for (int i = 0; i <= j; ++i) t += G.V[(int64_t)i * G.ld + e] * ys[i];
        x[e] = x[e] + t;
      });
}

// ---------------------------------------------------------------------------
// CG
// ---------------------------------------------------------------------------
enum { S_PQ = 3 };   // scal slot of the fused SpMV+dot result
// 1.0 while x += alpha p is pending: the update pass only moves r (reads r,
// q; writes r: 24 B/row) and the p pass, which reads p anyway, also moves x
// (reads x, r, p; writes x, p: 40 B/row) — 64 instead of 72 B/row of vector
// traffic per iteration.  The flag keeps the x update exactly once per
// iteration when a converged batch's later p passes are no-ops.
enum { S_XPEND = 4 };

// r = b - tmp; p = r; rr = r.r
__global__ void __launch_bounds__(KB) k_cg_restart(int64_t n, const double* __restrict__ b,
                                                   const double* __restrict__ t, double* __restrict__ r,
                                                   double* __restrict__ p, double* scal, double* partials,
                                                   unsigned* counter, svb_krylov_status* st) {
  double acc = 0.0;
  for_pairs(
      n,
      [&](int64_t e) {
        double2 bb = ld2(b + e), tt = ld2(t + e);
        double2 rr = make_double2(bb.x - tt.x, bb.y - tt.y);
        st2(r + e, rr);
        st2(p + e, rr);
        acc += rr.x * rr.x;
        acc += rr.y * rr.y;
      },
      [&](int64_t e) {
        double rr = b[e] - t[e];
        r[e] = rr;
        p[e] = rr;
        acc += rr * rr;
      });
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) {
    scal[S_RR] = tot;
    scal[S_XPEND] = 0.0;   // a restart starts from the current x
    st->beta = sqrt(tot);
    st->nonfinite = bad(tot);
  }
}

// Batched-CG control block (device memory): kernels of a batch become no-ops
// once `done` is set, so the host can enqueue many iterations and read the
// status once per batch; the estimate of every executed iteration is logged.
struct CgCtl {
  int done;       // CG_* reason, 0 while running
  int count;      // iterations executed since the last reset
  int cap;        // history capacity
  int pad;
  double tol;
  double* hist;   // per-iteration residual estimates
};
enum { CG_RUN = 0, CG_TOL = 1, CG_PQ0 = 2, CG_NONFINITE = 3 };

// r.r of the updated residual -> beta, rr, estimate, history, stop flags
__device__ __forceinline__ void cg_after_update(double* scal, double tot, double bnorm, svb_krylov_status* st,
                                                CgCtl* ctl) {
  const double rr_old = scal[S_RR];
  scal[S_BETA] = tot / rr_old;
  scal[S_RR] = tot;
  const double est = sqrt(tot) / bnorm;
  st->estimate = est;
  st->nonfinite = st->nonfinite || bad(tot) || bad(est);
  if (ctl != nullptr) {
    if (ctl->count < ctl->cap) ctl->hist[ctl->count] = est;
    ctl->count += 1;
    st->count = ctl->count;
    if (bad(tot) || bad(est)) ctl->done = CG_NONFINITE;
    else if (est <= ctl->tol) ctl->done = CG_TOL;
    st->done = ctl->done;
  }
}

// alpha = rr / (p.q)
__global__ void __launch_bounds__(KB) k_cg_pq(int64_t n, const double* __restrict__ p,
                                              const double* __restrict__ q, double* scal, double* partials,
                                              unsigned* counter, svb_krylov_status* st, CgCtl* ctl) {
  if (ctl != nullptr && ctl->done) return;
  double acc = 0.0;
  for_pairs(
      n,
      [&](int64_t e) {
        double2 a = ld2(p + e), c = ld2(q + e);
        acc += a.x * c.x;
        acc += a.y * c.y;
      },
      [&](int64_t e) { acc += p[e] * q[e]; });
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) {
    st->pq = tot;
    st->nonfinite = bad(tot);
    scal[S_ALPHA] = tot != 0.0 ? scal[S_RR] / tot : 0.0;
    if (ctl != nullptr && (bad(tot) || tot == 0.0)) {
      ctl->done = bad(tot) ? CG_NONFINITE : CG_PQ0;
      st->done = ctl->done;
    }
  }
}

// r -= alpha q; rr' = r.r; beta = rr'/rr; estimate; x += alpha p pending
// (applied by k_cg_p)
__global__ void __launch_bounds__(KB) k_cg_update(int64_t n, double* __restrict__ r, const double* __restrict__ q,
                                                  double* scal, double bnorm, double* partials,
                                                  unsigned* counter, svb_krylov_status* st, CgCtl* ctl) {
  if (ctl != nullptr && ctl->done) return;
  const double alpha = scal[S_ALPHA];
  double acc = 0.0;
  for_pairs(
      n,
      [&](int64_t e) {
        double2 rr = ld2(r + e), qq = ld2(q + e);
        rr.x -= alpha * qq.x;
        rr.y -= alpha * qq.y;
        st2(r + e, rr);
        acc += rr.x * rr.x;
        acc += rr.y * rr.y;
      },
      [&](int64_t e) {
        double rr = r[e] - alpha * q[e];
        r[e] = rr;
        acc += rr * rr;
      });
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) {
    scal[S_XPEND] = 1.0;
    cg_after_update(scal, tot, bnorm, st, ctl);
  }
}

// the same with alpha = rr / (p.q) from the fused DIA SpMV+dot
__global__ void __launch_bounds__(KB) k_cg_update_pq(int64_t n, double* __restrict__ r, const double* __restrict__ q,
                                                     double* scal, double bnorm, double* partials,
                                                     unsigned* counter, svb_krylov_status* st, CgCtl* ctl) {
  if (ctl->done) return;
  const double pq = scal[S_PQ];
  if (bad(pq) || pq == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->pq = pq;
      st->nonfinite = bad(pq);
      ctl->done = bad(pq) ? CG_NONFINITE : CG_PQ0;
      st->done = ctl->done;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st->pq = pq;
  const double alpha = scal[S_RR] / pq;
  double acc = 0.0;
  for_pairs(
      n,
      [&](int64_t e) {
        double2 rr = ld2(r + e), qq = ld2(q + e);
        rr.x -= alpha * qq.x;
        rr.y -= alpha * qq.y;
        st2(r + e, rr);
        acc += rr.x * rr.x;
        acc += rr.y * rr.y;
      },
      [&](int64_t e) {
        double rr = r[e] - alpha * q[e];
        r[e] = rr;
        acc += rr * rr;
      });
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) {
    scal[S_ALPHA] = alpha;
    scal[S_XPEND] = 1.0;
    cg_after_update(scal, tot, bnorm, st, ctl);
  }
}

// x += alpha p (when pending: once per update, even in the iteration that
// converged), then p = r + beta p unless the batch is done.  The last CTA
// to finish clears the pending flag (every CTA read it at its start).
__global__ void __launch_bounds__(KB) k_cg_p(int64_t n, double* __restrict__ x, const double* __restrict__ r,
                                             double* __restrict__ p, double* scal, const CgCtl* ctl,
                                             unsigned* counter) {
  const bool xmove = scal[S_XPEND] != 0.0;
  const bool pmove = !(ctl != nullptr && ctl->done);
  if (!xmove && !pmove) return;
  const double alpha = scal[S_ALPHA], beta = scal[S_BETA];
  for_pairs(
      n,
      [&](int64_t e) {
        const double2 pp = ld2(p + e);
        if (xmove) {
          const double2 xx = ld2(x + e);
          st2(x + e, make_double2(xx.x + alpha * pp.x, xx.y + alpha * pp.y));
        }
        if (pmove) {
          const double2 rr = ld2(r + e);
          st2(p + e, make_double2(rr.x + beta * pp.x, rr.y + beta * pp.y));
        }
      },
      [&](int64_t e) {
        const double pe = p[e];
        if (xmove) x[e] = x[e] + alpha * pe;
        if (pmove) p[e] = r[e] + beta * pe;
      });
  if (!xmove) return;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    scal[S_XPEND] = 0.0;
    *counter = 0;
  }
}

// ---------------------------------------------------------------------------
// building blocks for the row-partitioned solvers (device-scalar results)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(KB) k_axpy_dot(int64_t n, const double* __restrict__ alpha, double sign,
                                                 const double* __restrict__ x, double* __restrict__ y,
                                                 const double* __restrict__ z, double* partials,
                                                 unsigned* counter, double* out) {
  const double a = sign * (*alpha);
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double yy = y[e] + a * x[e];
    y[e] = yy;
    acc += (z ? z[e] : yy) * yy;
  }
  if (out == nullptr) return;
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) *out = tot;
}

__global__ void __launch_bounds__(KB) k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                                              double* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = a * x[e] + b * y[e];
}

__global__ void __launch_bounds__(KB) k_vscale(int64_t n, double* __restrict__ x, double s) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    x[e] *= s;
}

// generic dot for the host API
__global__ void __launch_bounds__(KB) k_dot(int64_t n, const double* __restrict__ a,
                                            const double* __restrict__ b, double* partials,
                                            unsigned* counter, double* out) {
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    acc += a[e] * b[e];
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) *out = tot;
}

// generic dot with an accumulate mode (row parts of one local SpMV)
__global__ void __launch_bounds__(KB) k_dot_acc(int64_t n, const double* __restrict__ a,
                                                const double* __restrict__ b, double* partials,
                                                unsigned* counter, double* out, int accumulate) {
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    acc += a[e] * b[e];
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) *out = accumulate ? *out + tot : tot;
}

// Row-partitioned CG on device scalars sc[] (all-reduced in place between
// the kernels), two vector passes per iteration after the SpMV+p.q pass:
//   k_dcg_rupdate: a = sc[icur]/sc[ipq] -> sc[ialpha], r -= a q, local r.r
//                  -> sc[out]  (reads r, q; writes r: 24 B/row)
//   k_dcg_xp:      x += a p, then p = r + b p with b = sc[inew]/sc[iold]
//                  (reads x, r, p; writes x, p: 40 B/row)
// i.e. the unfused x/r update + p update (48 + 24 B/row) regrouped so x
// moves in the pass that rewrites p, which reads p anyway.  A zero or
// non-finite p.Ap stores a = 0 and leaves r untouched (x then stays put too;
// the host confirms with the true residual or reports the breakdown) and
// copies r.r through unchanged.  Expressions are the contracted forms of
// the oracle loop's (oracle/cpu_oracle.py:cg): x + a p, r - a q, r + b p.
__global__ void __launch_bounds__(KB) k_dcg_rupdate(int64_t n, double* sc, int icur, int ipq, int out, int ialpha,
                                                    const double* __restrict__ q, double* __restrict__ r,
                                                    double* partials, unsigned* counter) {
  const double pq = sc[ipq];
  const bool ok = pq != 0.0 && isfinite(pq);
  const double a = ok ? sc[icur] / pq : 0.0;
  double acc = 0.0;
  if (ok && (((uintptr_t)q | (uintptr_t)r) & 15) != 0) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
      const double rn = r[e] - a * q[e];
      r[e] = rn;
      acc += rn * rn;
    }
  } else if (ok) {
    for_pairs(
        n,
        [&](int64_t e) {
          const double2 qq = ld2(q + e), rr = ld2(r + e);
          const double2 rn = make_double2(rr.x - a * qq.x, rr.y - a * qq.y);
          st2(r + e, rn);
          acc += rn.x * rn.x + rn.y * rn.y;
        },
        [&](int64_t e) {
          const double rn = r[e] - a * q[e];
          r[e] = rn;
          acc += rn * rn;
        });
  }
  double tot;
  if (grid_sum_last(acc, partials, counter, &tot) && threadIdx.x == 0) {
    sc[out] = ok ? tot : sc[icur];
    sc[ialpha] = a;
  }
}

__global__ void __launch_bounds__(KB) k_dcg_xp(int64_t n, const double* sc, int ialpha, int inew, int iold,
                                               const double* __restrict__ r, double* __restrict__ p,
                                               double* __restrict__ x) {
  const double a = sc[ialpha];
  const double b = sc[inew] / sc[iold];
  // p lives in a halo window at an odd element offset on some ranks: pairs
  // only when every operand is 16-byte aligned
  if ((((uintptr_t)r | (uintptr_t)p | (uintptr_t)x) & 15) != 0) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
      const double pe = p[e];
      x[e] = x[e] + a * pe;
      p[e] = r[e] + b * pe;
    }
    return;
  }
  for_pairs(
      n,
      [&](int64_t e) {
        const double2 rr = ld2(r + e), pp = ld2(p + e), xx = ld2(x + e);
        st2(x + e, make_double2(xx.x + a * pp.x, xx.y + a * pp.y));
        st2(p + e, make_double2(rr.x + b * pp.x, rr.y + b * pp.y));
      },
      [&](int64_t e) {
        const double pe = p[e];
        x[e] = x[e] + a * pe;
        p[e] = r[e] + b * pe;
      });
}

// ---------------------------------------------------------------------------
// Row-partitioned GMRES: classical Gram-Schmidt twice (CGS2) over a block of
// basis rows V[r0 .. r0+k) (row stride ld, k <= VB), so an Arnoldi step needs
// two all-reduces across ranks instead of MGS's j+2:
//   GS_DOT:    out[i] = V_i . w
//   GS_UPDATE: w -= sum_i h[i] V_i; out[i] = V_i . w; out[k] = w . w
//   GS_FINISH: dst = (w - sum_i h[i] V_i) / *div
//   GS_AXPY:   dst = w + sum_i h[i] V_i          (x += V y at a restart)
// Each basis row is loaded once per element (registers), the k(+1) sums are
// folded per CTA and, by the last CTA to finish, in fixed CTA order.
// ---------------------------------------------------------------------------
constexpr int VB = 32;
enum { GS_DOT = 0, GS_UPDATE = 1, GS_FINISH = 2, GS_AXPY = 3 };   // C-ABI modes
enum { K_DOT = 0, K_UPDATE = 1, K_SUB = 2, K_ADD = 3 };            // kernel modes

// K_DOT:    out[i] = V_i . w (+ out[k] = w . w with `norm`)
// K_UPDATE: t = w - sum h_i V_i -> dst; out[i] = V_i . t; out[k] = t . t
// K_SUB:    dst = (w - sum h_i V_i) [/ *div]
// K_ADD:    dst = w + sum h_i V_i
template <int MODE>
__global__ void __launch_bounds__(KB) k_gs_block(int64_t n, const double* __restrict__ V, int64_t ld, int k,
                                                 const double* __restrict__ h, const double* __restrict__ div,
                                                 int norm, const double* w, double* dst, double* partials,
                                                 unsigned* counter, double* out) {
  constexpr bool DOTS = MODE == K_DOT || MODE == K_UPDATE;
  constexpr int NS = DOTS ? VB + 1 : 1;
  __shared__ double hs[VB];
  __shared__ double red[KB / 32][VB + 1];
  __shared__ bool last;
  if (MODE != K_DOT && threadIdx.x < k) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  const bool scale = MODE == K_SUB && div != nullptr;
  const double dv = scale ? *div : 1.0;
  double acc[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) acc[i] = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double v[VB];
#pragma unroll
    for (int i = 0; i < VB; ++i)
      if (i < k) v[i] = __ldcs(V + (int64_t)i * ld + e);
    double t = w[e];
    if (MODE == K_UPDATE || MODE == K_SUB) {
#pragma unroll
      for (int i = 0; i < VB; ++i)
        if (i < k) t -= hs[i] * v[i];
    } else if (MODE == K_ADD) {
#pragma unroll
      for (int i = 0; i < VB; ++i)
        if (i < k) t += hs[i] * v[i];
    }
    if (scale) t = t / dv;
    if (MODE != K_DOT) dst[e] = t;
    if (DOTS) {
#pragma unroll
      for (int i = 0; i < VB; ++i)
        if (i < k) acc[i] += v[i] * t;
      if (norm) acc[VB] += t * t;
    }
  }
  if (!DOTS) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nv = k + (norm ? 1 : 0);
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    if (i < k || (i == VB && norm)) {
      double a = acc[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) red[wid][i < VB ? i : k] = a;   // the norm lands right after the k dots
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double b = 0.0;
    for (int q = 0; q < KB / 32; ++q) b += red[q][threadIdx.x];
    partials[(int64_t)blockIdx.x * (VB + 1) + threadIdx.x] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < nv) {
    double t = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(partials + (int64_t)b * (VB + 1) + threadIdx.x);
    out[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) *counter = 0;
}

// hn = sqrt(max(nrm - sum h2_i^2, 0)): ||w2|| of the second CGS pass from
// ||w1||^2 and the (tiny) re-orthogonalisation coefficients (w2 = w1 - V h2
// with V orthonormal), so no third reduction is needed
__global__ void k_gs_hn(const double* __restrict__ h2, int k, const double* __restrict__ nrm, double* hn) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < k; ++i) s += h2[i] * h2[i];
  const double r = *nrm - s;
  *hn = r > 0.0 ? sqrt(r) : 0.0;
}

__global__ void __launch_bounds__(KB) k_fill(double* __restrict__ x, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

static Gm gm_of(svb_krylov* k) {
  Gm G;
  G.V = ptr<double>(k->V);
  G.n = k->n;
  G.ld = k->ld;
  G.m = k->m;
  G.H = ptr<double>(k->H);
  G.cs = ptr<double>(k->cs);
  G.sn = ptr<double>(k->sn);
  G.g = ptr<double>(k->g);
  G.y = ptr<double>(k->y);
  G.partials = ptr<double>(k->partials);
  G.counter = ptr<unsigned>(k->counter);
  G.st = k->st_dev;
  return G;
}

}  // namespace svb

using namespace svb;

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// CTAs of the TMA Arnoldi kernel.  Every MGS pass ends in a grid-wide
// exchange whose latency grows with the number of CTAs taking part, while a
// small basis is L2-resident and cheap to stream from few SMs: small systems
// run on fewer CTAs, one per 4096 rows (two ring chunks), at least 32.
// Measured per GMRES(30) iteration (profiles/r2_mgs_grid_ab.json, G = 148 ->
// this rule): n = 65 K 70.9 -> 50.3 us, 131 K 72.8 -> 57.7, 262 K 77.4 ->
// 63.9; from n = 606 K on all 148 SMs take part as before.
// SPMVTUNE_MGS_GRID overrides (A/B runs).
static int mgs_grid(int64_t n, int sms) {
  int g = (int)std::min<int64_t>(sms, std::max<int64_t>(32, (n + 4095) / 4096));
  if (const char* e = std::getenv("SPMVTUNE_MGS_GRID")) {
    const int v = std::atoi(e);
    if (v >= 1 && v <= sms) g = v;
  }
  return std::min<int>(sms, std::max<int>(g, (int)((n + svb::mgs::MAX_SLICE - 1) / svb::mgs::MAX_SLICE)));
}

extern "C" {

int svb_krylov_create(int64_t n, int32_t m, svb_krylov** out) {
  return guard([&] {
    SVB_REQUIRE(n >= 1 && m >= 0 && m <= KRYLOV_MAX_M, SVB_INVALID,
                "krylov workspace: n >= 1, 0 <= restart m <= 24000");
    cudaStream_t s = 0;
    auto k = new svb_krylov();
    k->n = n;
    k->m = m;
    k->ld = (n + 31) & ~int64_t(31);  // 256-byte aligned rows
    k->rgrid = grid_for(n / 2 + 1, KB, 4);
    const int64_t mm = m > 0 ? m : 1;
    k->V = alloc((m + 1) * k->ld * 8, s);
    k->x = alloc(k->ld * 8, s);
    k->b = alloc(k->ld * 8, s);
    k->tmp = alloc(k->ld * 8, s);
    k->p = alloc(k->ld * 8, s);
    k->q = alloc(k->ld * 8, s);
    k->r = alloc(k->ld * 8, s);
    k->H = alloc((mm + 1) * mm * 8, s);
    k->cs = alloc(mm * 8, s);
    k->sn = alloc(mm * 8, s);
    k->g = alloc((mm + 1) * 8, s);
    k->y = alloc(mm * 8, s);
    k->scal = alloc(8 * 8, s);
    SVB_CUDA_TRY(cudaMemsetAsync(k->scal->ptr, 0, 8 * 8, s));   // S_XPEND = 0
    k->partials = alloc(k->rgrid * 8, s);
    k->counter = alloc(8, s);
    SVB_CUDA_TRY(cudaMemsetAsync(k->counter->ptr, 0, 8, s));
    SVB_CUDA_TRY(cudaMemsetAsync(k->x->ptr, 0, k->ld * 8, s));
    // SM-resident MGS when every CTA's slice of w fits in shared memory
    {
      int dev = 0, optin = 0, coop = 0;
      SVB_CUDA_TRY(cudaGetDevice(&dev));
      SVB_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      SVB_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
      const int G = sm_count();
      k->chunk = (((n + G - 1) / G) + 1) & ~int64_t(1);
      k->res_smem = (size_t)(k->chunk + 34) * sizeof(double);
      const char* mode = std::getenv("SPMVTUNE_MGS");
      const bool allowed = !(mode && std::strcmp(mode, "stream") == 0);
      // TMA-streamed MGS: w in registers + smem, V_{i-1} in TMEM, the basis
      // rows streamed once through a bulk-copy ring; slices above the
      // on-chip capacity (mgs::MAX_SLICE = 32768 doubles: n > 4.85 M on 148
      // SMs) run partially resident up to n = 19.4 M (mgs::plan)
      const bool tma_ok = !(mode && (std::strcmp(mode, "resident") == 0 || std::strcmp(mode, "tmem") == 0)) &&
                          m + 2 < 255;
      k->tma_grid = mgs_grid(n, G);
      k->tma_chunk = (((n + k->tma_grid - 1) / k->tma_grid) + 1) & ~int64_t(1);
      if (allowed && coop && m >= 1 && tma_ok &&
          mgs::plan(k->tma_chunk, &k->tma_chunks, &k->tma_stages, &k->tma_nres) &&
          mgs::SMEM <= (size_t)optin) {
        const void* kern = k->tma_nres < k->tma_chunks ? (const void*)mgs::k_mgs_tma<true>
                                                       : (const void*)mgs::k_mgs_tma<false>;
        SVB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mgs::SMEM));
        int per = 0;
        SVB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, mgs::NT, mgs::SMEM));
        if (per >= 1) {
          k->tma = true;
          const size_t gb = 2 * (size_t)mgs::SLOT_STRIDE * G * sizeof(unsigned long long);
          k->gslot = alloc(gb, s);
          SVB_CUDA_TRY(cudaMemsetAsync(k->gslot->ptr, 0, gb, s));
        }
      }
      if (allowed && coop && m >= 1 && k->res_smem <= (size_t)optin) {
        SVB_CUDA_TRY(cudaFuncSetAttribute(k_gm_mgs_resident, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)k->res_smem));
        int per_sm = 0;
        SVB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gm_mgs_resident, PB,
                                                                   k->res_smem));
        k->resident = per_sm >= 1;
        k->gparts = alloc(2 * G * sizeof(double) + 64, s);   // + grid counter
        // TMEM-staged variant: every thread parks up to 32 doubles of V_i in
        // TMEM; at least 120 KB of dynamic smem keeps one CTA per SM so the
        // full 512-column TMEM allocation can never contend
        const bool tmem_ok = !(mode && std::strcmp(mode, "resident") == 0) &&
                             (k->chunk + PB - 1) / PB <= TMEM_MAX_PER_THREAD;
        if (k->resident && tmem_ok) {
          k->tmem_smem = std::max<size_t>(k->res_smem, 120 * 1024);
          if (k->tmem_smem <= (size_t)optin) {
            SVB_CUDA_TRY(cudaFuncSetAttribute(k_gm_mgs_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)k->tmem_smem));
            int per = 0;
            SVB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gm_mgs_tmem, PB, k->tmem_smem));
            k->tmem = per == 1;
          }
        }
      }
    }
    SVB_CUDA_TRY(cudaEventCreateWithFlags(&k->ev, cudaEventDisableTiming));
    SVB_CUDA_TRY(cudaHostAlloc((void**)&k->st_host, sizeof(svb_krylov_status), cudaHostAllocMapped));
    std::memset(k->st_host, 0, sizeof(svb_krylov_status));
    SVB_CUDA_TRY(cudaHostGetDevicePointer((void**)&k->st_dev, k->st_host, 0));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = k;
  });
}

int svb_krylov_destroy(svb_krylov* k) {
  return guard([&] {
    SVB_CUDA_TRY(cudaDeviceSynchronize());
    delete k;
  });
}

int svb_krylov_vec(svb_krylov* k, int which, double** out) {
  return guard([&] {
    SVB_REQUIRE(k && out, SVB_INVALID, "null workspace");
    if (which >= 0) {
      SVB_REQUIRE(which <= k->m, SVB_INVALID, "V row out of range");
      *out = ptr<double>(k->V) + (int64_t)which * k->ld;
      return;
    }
    switch (which) {
      case -1: *out = ptr<double>(k->x); break;
      case -2: *out = ptr<double>(k->b); break;
      case -3: *out = ptr<double>(k->tmp); break;
      case -4: *out = ptr<double>(k->p); break;
      case -5: *out = ptr<double>(k->q); break;
      case -6: *out = ptr<double>(k->r); break;
      default: throw Error{SVB_INVALID, "unknown workspace vector"};
    }
  });
}

static void mark(svb_krylov* k, cudaStream_t s) { SVB_CUDA_TRY(cudaEventRecord(k->ev, s)); }

int svb_krylov_mark(svb_krylov* k, void* stream) {
  return guard([&] { mark(k, S(stream)); });
}

int svb_krylov_status_get(svb_krylov* k, void* stream, svb_krylov_status* out) {
  return guard([&] {
    (void)stream;
    SVB_CUDA_TRY(cudaEventSynchronize(k->ev));
    std::atomic_thread_fence(std::memory_order_seq_cst);
    std::memcpy(out, (const void*)k->st_host, sizeof(svb_krylov_status));
  });
}

int svb_krylov_bnorm(svb_krylov* k, void* stream) {
  return guard([&] {
    k_resnorm<<<k->rgrid, KB, 0, S(stream)>>>(ptr<double>(k->b), nullptr, k->n, ptr<double>(k->partials),
                                               ptr<unsigned>(k->counter), k->st_dev);
    SVB_CHECK_LAUNCH();
    mark(k, S(stream));
  });
}

int svb_krylov_residual(svb_krylov* k, void* stream) {
  return guard([&] {
    k_resnorm<<<k->rgrid, KB, 0, S(stream)>>>(ptr<double>(k->b), ptr<double>(k->tmp), k->n,
                                               ptr<double>(k->partials), ptr<unsigned>(k->counter),
                                               k->st_dev);
    SVB_CHECK_LAUNCH();
    mark(k, S(stream));
  });
}

int svb_gmres_restart(svb_krylov* k, void* stream) {
  return guard([&] {
    SVB_REQUIRE(k->m >= 1, SVB_INVALID, "GMRES workspace needs restart m >= 1");
    k->normalized = -1;
    Gm G = gm_of(k);
    cudaStream_t s = S(stream);
    const size_t mm = (size_t)k->m;
    SVB_CUDA_TRY(cudaMemsetAsync(G.H, 0, (mm + 1) * mm * 8, s));
    SVB_CUDA_TRY(cudaMemsetAsync(G.cs, 0, mm * 8, s));
    SVB_CUDA_TRY(cudaMemsetAsync(G.sn, 0, mm * 8, s));
    SVB_CUDA_TRY(cudaMemsetAsync(G.g, 0, (mm + 1) * 8, s));
    k_gm_residual<<<k->rgrid, KB, 0, S(stream)>>>(G, ptr<double>(k->b), ptr<double>(k->tmp));
    SVB_CHECK_LAUNCH();
    mark(k, S(stream));
    k_gm_scale<<<k->rgrid, KB, 0, S(stream)>>>(G.V, k->n, G.g);
    SVB_CHECK_LAUNCH();
  });
}

int svb_gmres_arnoldi(svb_krylov* k, int32_t j, double bnorm, void* stream) {
  return guard([&] {
    SVB_REQUIRE(j >= 0 && j < k->m, SVB_INVALID, "Arnoldi column out of range");
    Gm G = gm_of(k);
    cudaStream_t s = S(stream);
    if (k->tma) {
      mgs::Args A{};
      A.V = G.V;
      A.n = G.n;
      A.ld = G.ld;
      A.chunk = k->tma_chunk;
      A.m = G.m;
      A.j = j;
      A.H = G.H;
      A.cs = G.cs;
      A.sn = G.sn;
      A.g = G.g;
      A.st = G.st;
      A.bnorm = bnorm;
      A.gslot = ptr<unsigned long long>(k->gslot);
      A.epoch = ++k->epoch;
      A.chunk_count = k->tma_chunks;
      A.nsb = k->tma_stages;
      A.nres = k->tma_nres;
      A.trace = nullptr;
      void* args[] = {&A};
      const void* kern = k->tma_nres < k->tma_chunks ? (const void*)mgs::k_mgs_tma<true>
                                                     : (const void*)mgs::k_mgs_tma<false>;
      SVB_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3(k->tma_grid), dim3(mgs::NT), args, mgs::SMEM, s));
      note_launches(1);
      k->normalized = j;
      mark(k, s);
      return;
    }
    if (k->resident) {
      int64_t chunk = k->chunk;
      double* gp = ptr<double>(k->gparts);
      unsigned* gc = reinterpret_cast<unsigned*>(gp + 2 * sm_count());
      SVB_CUDA_TRY(cudaMemsetAsync(gc, 0, sizeof(unsigned), s));
      void* args[] = {&G, &j, &bnorm, &chunk, &gp, &gc};
      if (k->tmem)
        SVB_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_gm_mgs_tmem, dim3(sm_count()), dim3(PB), args,
                                                 k->tmem_smem, s));
      else
        SVB_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_gm_mgs_resident, dim3(sm_count()), dim3(PB),
                                                 args, k->res_smem, s));
      note_launches(1);
      k->normalized = j;
      mark(k, s);
      return;
    }
    k->normalized = -1;
    k_gm_dot0<<<k->rgrid, KB, 0, s>>>(G, j);
    for (int i = 1; i <= j; ++i) k_gm_pass<<<k->rgrid, KB, 0, s>>>(G, i, j);
    k_gm_final<<<k->rgrid, KB, 0, s>>>(G, j, bnorm);
    note_launches(j + 1);
    SVB_CHECK_LAUNCH();
    mark(k, s);
  });
}

int svb_gmres_normalize(svb_krylov* k, int32_t j, void* stream) {
  return guard([&] {
    if (k->normalized == j) return;  // already done (resident MGS kernel or an earlier call)
    Gm G = gm_of(k);
    k_gm_scale<<<k->rgrid, KB, 0, S(stream)>>>(G.V + (int64_t)(j + 1) * G.ld, k->n, G.H + (j + 1) * G.m + j);
    SVB_CHECK_LAUNCH();
    k->normalized = j;
  });
}

int svb_gmres_update_x(svb_krylov* k, int32_t j, void* stream) {
  return guard([&] {
    SVB_REQUIRE(j >= 0 && j < k->m, SVB_INVALID, "Arnoldi column out of range");
    Gm G = gm_of(k);
    const int nj = j + 1;
    size_t dyn = 32 * sizeof(double);
    if (nj > 32) {
      k_gm_solve_y<<<1, 32, 0, S(stream)>>>(G, j);
      SVB_CHECK_LAUNCH();
      dyn = (size_t)nj * sizeof(double);
      // opt in to the dynamic smem range (per device; a cheap host call)
      SVB_CUDA_TRY(cudaFuncSetAttribute(k_gm_update_x, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(KRYLOV_MAX_M * sizeof(double) + 8)));
    }
    k_gm_update_x<<<k->rgrid, KB, dyn, S(stream)>>>(G, j, ptr<double>(k->x));
    SVB_CHECK_LAUNCH();
  });
}

int svb_cg_restart(svb_krylov* k, void* stream) {
  return guard([&] {
    k_cg_restart<<<k->rgrid, KB, 0, S(stream)>>>(k->n, ptr<double>(k->b), ptr<double>(k->tmp), ptr<double>(k->r),
                                                  ptr<double>(k->p), ptr<double>(k->scal), ptr<double>(k->partials),
                                                  ptr<unsigned>(k->counter), k->st_dev);
    SVB_CHECK_LAUNCH();
    mark(k, S(stream));
  });
}

int svb_cg_step(svb_krylov* k, double bnorm, void* stream) {
  return guard([&] {
    cudaStream_t s = S(stream);
    double* P = ptr<double>(k->partials);
    unsigned* C = ptr<unsigned>(k->counter);
    k_cg_pq<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->p), ptr<double>(k->q), ptr<double>(k->scal), P, C,
                                     k->st_dev, nullptr);
    k_cg_update<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->r), ptr<double>(k->q), ptr<double>(k->scal), bnorm, P,
                                         C, k->st_dev, nullptr);
    mark(k, s);  // status is final here; the x/p pass overlaps the host
    k_cg_p<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->x), ptr<double>(k->r), ptr<double>(k->p),
                                    ptr<double>(k->scal), nullptr, C);
    note_launches(2);
    SVB_CHECK_LAUNCH();
  });
}

int svb_cg_batch_reset(svb_krylov* k, double tol, int64_t cap, void* stream) {
  return guard([&] {
    cudaStream_t s = S(stream);
    if (cap < 1) cap = 1;
    if (!k->hist || k->hist_cap < cap) {
      k->hist = alloc(cap * sizeof(double), s);
      detach(k->hist);
      k->hist_cap = cap;
    }
    if (!k->ctl) {
      k->ctl = alloc(sizeof(CgCtl), s);
      detach(k->ctl);
    }
    CgCtl c{CG_RUN, 0, (int)std::min<int64_t>(k->hist_cap, INT32_MAX), 0, tol, ptr<double>(k->hist)};
    SVB_CUDA_TRY(cudaMemcpyAsync(k->ctl->ptr, &c, sizeof(c), cudaMemcpyHostToDevice, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));   // `c` is a host temporary
    k->st_host->done = 0;
    k->st_host->count = 0;
  });
}

int svb_cg_batch_resume(svb_krylov* k, void* stream) {
  return guard([&] {
    SVB_REQUIRE(k->ctl, SVB_INVALID, "svb_cg_batch_reset first");
    SVB_CUDA_TRY(cudaMemsetAsync(k->ctl->ptr, 0, sizeof(int), S(stream)));   // done = 0
    SVB_CUDA_TRY(cudaStreamSynchronize(S(stream)));
    k->st_host->done = 0;
  });
}

int svb_cg_step_batched(svb_krylov* k, double bnorm, void* stream) {
  return guard([&] {
    SVB_REQUIRE(k->ctl, SVB_INVALID, "svb_cg_batch_reset first");
    cudaStream_t s = S(stream);
    double* P = ptr<double>(k->partials);
    unsigned* C = ptr<unsigned>(k->counter);
    CgCtl* ctl = ptr<CgCtl>(k->ctl);
    k_cg_pq<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->p), ptr<double>(k->q), ptr<double>(k->scal), P, C,
                                     k->st_dev, ctl);
    k_cg_update<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->r), ptr<double>(k->q), ptr<double>(k->scal), bnorm, P,
                                         C, k->st_dev, ctl);
    k_cg_p<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->x), ptr<double>(k->r), ptr<double>(k->p),
                                    ptr<double>(k->scal), ctl, C);
    note_launches(2);
    SVB_CHECK_LAUNCH();
    mark(k, s);
  });
}

int svb_cg_step_batched_dia(svb_krylov* k, const svb_matrix* m, double bnorm, void* stream) {
  return guard([&] {
    SVB_REQUIRE(k->ctl, SVB_INVALID, "svb_cg_batch_reset first");
    SVB_REQUIRE(m && m->fmt == SVB_DIA && m->nrows == k->n && m->ncols == k->n, SVB_DIM_MISMATCH,
                "fused CG step needs the square DIA operator of this workspace");
    cudaStream_t s = S(stream);
    double* P = ptr<double>(k->partials);
    unsigned* C = ptr<unsigned>(k->counter);
    CgCtl* ctl = ptr<CgCtl>(k->ctl);
    double* sc = ptr<double>(k->scal);
    if (!k->dparts) {
      k->dgrid = grid_for(k->n, 256, 8);
      k->dparts = alloc(k->dgrid * 8 + 64, s);
      detach(k->dparts);   // long-lived: freed on the legacy stream, not this thread's
      SVB_CUDA_TRY(cudaMemsetAsync(ptr<double>(k->dparts) + k->dgrid, 0, 64, s));
    }
    launch_dia_dot(m, ptr<double>(k->p), ptr<double>(k->q), ptr<double>(k->p), ptr<double>(k->dparts),
                   reinterpret_cast<unsigned*>(ptr<double>(k->dparts) + k->dgrid), sc + S_PQ, &ctl->done,
                   k->dgrid, s);
    k_cg_update_pq<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->r), ptr<double>(k->q), sc, bnorm, P, C, k->st_dev,
                                            ctl);
    SVB_CHECK_LAUNCH();
    k_cg_p<<<k->rgrid, KB, 0, s>>>(k->n, ptr<double>(k->x), ptr<double>(k->r), ptr<double>(k->p), sc, ctl, C);
    SVB_CHECK_LAUNCH();
    mark(k, s);
  });
}

int svb_cg_history(svb_krylov* k, int64_t first, int64_t count, double* host, void* stream) {
  return guard([&] {
    SVB_REQUIRE(k->hist && first >= 0 && first + count <= k->hist_cap, SVB_INVALID, "history range");
    if (count <= 0) return;
    SVB_CUDA_TRY(cudaMemcpyAsync(host, ptr<double>(k->hist) + first, count * sizeof(double),
                                 cudaMemcpyDeviceToHost, S(stream)));
    SVB_CUDA_TRY(cudaStreamSynchronize(S(stream)));
  });
}

int svb_vecops_create(int64_t n, svb_vecops** out) {
  return guard([&] {
    auto v = new svb_vecops();
    v->n = n;
    v->grid = grid_for(n, KB, 4);
    v->partials = alloc(v->grid * 8 + 64, 0);
    detach(v->partials);
    SVB_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(v->partials->ptr) + v->grid * 8, 0, 64, 0));

    SVB_CUDA_TRY(cudaStreamSynchronize(0));
    *out = v;
  });
}

int svb_vecops_destroy(svb_vecops* v) {
  return guard([&] {
    SVB_CUDA_TRY(cudaDeviceSynchronize());
    delete v;
  });
}

static unsigned* vctr(svb_vecops* v) {
  return reinterpret_cast<unsigned*>(static_cast<char*>(v->partials->ptr) + v->grid * 8);
}

int svb_vec_dot(svb_vecops* v, const double* x, const double* y, double* out, void* stream) {
  return guard([&] {
    k_dot<<<v->grid, KB, 0, S(stream)>>>(v->n, x, y, ptr<double>(v->partials), vctr(v), out);
    SVB_CHECK_LAUNCH();
  });
}

int svb_vec_axpy_dot(svb_vecops* v, const double* alpha, double sign, const double* x, double* y,
                     const double* z, double* out, void* stream) {
  return guard([&] {
    k_axpy_dot<<<v->grid, KB, 0, S(stream)>>>(v->n, alpha, sign, x, y, z, ptr<double>(v->partials), vctr(v),
                                               out);
    SVB_CHECK_LAUNCH();
  });
}

static double* bpart(svb_vecops* v, unsigned** ctr) {
  if (!v->bpart) {
    v->bpart = alloc((size_t)v->grid * (VB + 1) * 8 + 64, 0);
    detach(v->bpart);
    SVB_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(v->bpart->ptr) + (size_t)v->grid * (VB + 1) * 8, 0, 64, 0));
    SVB_CUDA_TRY(cudaStreamSynchronize(0));
  }
  *ctr = reinterpret_cast<unsigned*>(static_cast<char*>(v->bpart->ptr) + (size_t)v->grid * (VB + 1) * 8);
  return ptr<double>(v->bpart);
}

// rows [0, k) of V in groups of at most VB per launch
int svb_vec_gs(svb_vecops* v, int32_t mode, const double* V, int64_t ld, int32_t k, const double* h,
               const double* div, const double* w, double* dst, double* out, void* stream) {
  return guard([&] {
    SVB_REQUIRE(k >= 1 && V && w, SVB_INVALID, "block Gram-Schmidt: k >= 1 rows and w required");
    SVB_REQUIRE(mode >= GS_DOT && mode <= GS_AXPY, SVB_INVALID, "block Gram-Schmidt: unknown mode");
    SVB_REQUIRE(mode == GS_DOT || (h && dst), SVB_INVALID, "block Gram-Schmidt: coefficients and dst required");
    SVB_REQUIRE(!(mode == GS_DOT || mode == GS_UPDATE) || out, SVB_INVALID, "block Gram-Schmidt: output required");
    SVB_REQUIRE(mode != GS_FINISH || div, SVB_INVALID, "block Gram-Schmidt: divisor required");
    if (v->n == 0) {   // a rank without rows still produces its (zero) partials
      if (mode == GS_DOT || mode == GS_UPDATE)
        SVB_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)(k + (mode == GS_UPDATE)) * 8, S(stream)));
      return;
    }
    cudaStream_t s = S(stream);
    unsigned* ctr = nullptr;
    double* part = bpart(v, &ctr);
    auto row = [&](int g) { return V + (int64_t)g * ld; };
    if (mode == GS_UPDATE && k <= VB) {   // fused: one pass
      k_gs_block<K_UPDATE><<<v->grid, KB, 0, s>>>(v->n, V, ld, k, h, nullptr, 1, w, dst, part, ctr, out);
      SVB_CHECK_LAUNCH();
      return;
    }
    const double* src = w;
    if (mode != GS_DOT) {   // apply the coefficients group by group (in row order)
      for (int g = 0; g < k; g += VB) {
        const int kk = std::min(VB, k - g);
        const bool lastg = g + kk >= k;
        if (mode == GS_AXPY)
          k_gs_block<K_ADD><<<v->grid, KB, 0, s>>>(v->n, row(g), ld, kk, h + g, nullptr, 0, src, dst, part, ctr,
                                                   nullptr);
        else
          k_gs_block<K_SUB><<<v->grid, KB, 0, s>>>(v->n, row(g), ld, kk, h + g,
                                                   (mode == GS_FINISH && lastg) ? div : nullptr, 0, src, dst,
                                                   part, ctr, nullptr);
        SVB_CHECK_LAUNCH();
        src = dst;
      }
      if (mode != GS_UPDATE) return;
    }
    // dots of the (updated) w against every row; the norm with the last group
    for (int g = 0; g < k; g += VB) {
      const int kk = std::min(VB, k - g);
      const int nrm = (mode == GS_UPDATE && g + kk >= k) ? 1 : 0;
      k_gs_block<K_DOT><<<v->grid, KB, 0, s>>>(v->n, row(g), ld, kk, nullptr, nullptr, nrm, src, nullptr, part,
                                               ctr, out + g);
      SVB_CHECK_LAUNCH();
    }
  });
}

int svb_vec_gs_hn(const double* h2, int32_t k, const double* nrm, double* hn, void* stream) {
  return guard([&] {
    k_gs_hn<<<1, 32, 0, S(stream)>>>(h2, k, nrm, hn);
    SVB_CHECK_LAUNCH();
  });
}

int svb_vec_spmv_dot(svb_vecops* v, const svb_matrix* m, int format, int library, int lane, int workers,
                     const double* x, double* y, const double* dsrc, double* out, int32_t accumulate, void* stream) {
  return guard([&] {
    SVB_REQUIRE(m && out, SVB_INVALID, "null argument");
    cudaStream_t s = S(stream);
    if (!v->spart) {
      v->sgrid = std::max<unsigned>(grid_for(std::max<int64_t>(v->n, 1), 256, 8), (unsigned)sm_count());
      v->spart = alloc((size_t)v->sgrid * 8 + 64, 0);
      detach(v->spart);
      SVB_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(v->spart->ptr) + (size_t)v->sgrid * 8, 0, 64, 0));
      SVB_CUDA_TRY(cudaStreamSynchronize(0));
    }
    double* part = ptr<double>(v->spart);
    unsigned* ctr = reinterpret_cast<unsigned*>(static_cast<char*>(v->spart->ptr) + (size_t)v->sgrid * 8);
    if (m->nrows == 0) {
      if (!accumulate) SVB_CUDA_TRY(cudaMemsetAsync(out, 0, 8, s));
      return;
    }
    if (format == SVB_DIA && m->fmt == SVB_DIA && grid_for(m->nrows, 256, 8) <= v->sgrid) {
      launch_dia_dot(m, x, y, dsrc, part, ctr, out, nullptr, v->sgrid, s, accumulate);
      return;
    }
    spmv_dispatch(m, format, library, lane, workers, SVB_F64, x, y, s);
    k_dot_acc<<<grid_for(m->nrows, KB, 4), KB, 0, s>>>(m->nrows, dsrc, y, part, ctr, out, accumulate);
    SVB_CHECK_LAUNCH();
  });
}

int svb_dcg_rupdate(svb_vecops* v, double* sc, int32_t icur, int32_t ipq, int32_t out, int32_t ialpha,
                    const double* q, double* r, void* stream) {
  return guard([&] {
    k_dcg_rupdate<<<v->grid, KB, 0, S(stream)>>>(v->n, sc, icur, ipq, out, ialpha, q, r, ptr<double>(v->partials),
                                                  vctr(v));
    SVB_CHECK_LAUNCH();
  });
}

int svb_dcg_xp(svb_vecops* v, const double* sc, int32_t ialpha, int32_t inew, int32_t iold, const double* r,
               double* p, double* x, void* stream) {
  return guard([&] {
    k_dcg_xp<<<v->grid, KB, 0, S(stream)>>>(v->n, sc, ialpha, inew, iold, r, p, x);
    SVB_CHECK_LAUNCH();
  });
}

int svb_vec_axpby(svb_vecops* v, double a, const double* x, double b, double* y, void* stream) {
  return guard([&] {
    k_axpby<<<v->grid, KB, 0, S(stream)>>>(v->n, a, x, b, y);
    SVB_CHECK_LAUNCH();
  });
}

int svb_vec_scale(svb_vecops* v, double* x, double s, void* stream) {
  return guard([&] {
    k_vscale<<<v->grid, KB, 0, S(stream)>>>(v->n, x, s);
    SVB_CHECK_LAUNCH();
  });
}

int svb_fill(double* x, int64_t n, double v, void* stream) {
  return guard([&] {
    if (n <= 0) return;
    k_fill<<<grid_for(n, KB), KB, 0, S(stream)>>>(x, n, v);
    SVB_CHECK_LAUNCH();
  });
}

int svb_dot(const double* x, const double* y, int64_t n, double* out_host, void* stream) {
  return guard([&] {
    cudaStream_t s = S(stream);
    const unsigned g = grid_for(n, KB, 4);
    Buf part = alloc(g * 8 + 16, s);
    unsigned* ctr = reinterpret_cast<unsigned*>(static_cast<char*>(part->ptr) + g * 8);
    double* res = reinterpret_cast<double*>(static_cast<char*>(part->ptr) + g * 8 + 8);
    SVB_CUDA_TRY(cudaMemsetAsync(ctr, 0, 4, s));
    k_dot<<<g, KB, 0, s>>>(n, x, y, ptr<double>(part), ctr, res);
    SVB_CHECK_LAUNCH();
    SVB_CUDA_TRY(cudaMemcpyAsync(out_host, res, 8, cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
