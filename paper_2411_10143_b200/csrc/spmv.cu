// The 13 SpMV configurations of the reference (kernels.py:146-312) as sm_100a
// kernels, fp64 and fp32.
//
// Numerics: this translation unit is compiled with -fmad=false, so every
// product v*x[c] is rounded before it is added, exactly like numpy.  Each
// deterministic kernel reproduces the reference's summation order, which
// makes the fp64 results bit-identical to the CPU path:
//   CSR/LibA/L   lane j%L sequential from 0, halving tree  -> warp shuffles
//   CSR/LibB     p[s] + pairwise(p[s+1:e])                -> staged row segments
//   CSR/LibC     per (row x chunk) segment, chunk order    -> staged row pieces
//   COO/LibA     reduceat over row runs                    -> tile segmented reduce
//   COO/LibB     np.add.at, random order                   -> warp-aggregated atomics
//   ELL/LibA     column sweep from 0                       -> thread per row
//   ELL/LibC     S strided partials, merged in order       -> thread per row
//   DIA/LibA     ascending-offset sweep                    -> thread per row
//   HYB/LibA     ELL sweep, then += reduceat(spill)        -> two kernels
// All kernels are bandwidth-bound (~2 flop per 12-16 B): no tensor cores.
#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "matrix.cuh"

namespace svb {

constexpr int ROWSEG_ROWS = 128;     // rows per CTA of the staged row-segment kernel
constexpr int ROWSEG_CAP = 2048;     // staged products per CTA
constexpr int COO_THREADS = 128;
constexpr int COO_ITEMS = 8;
constexpr int COO_TILE = COO_THREADS * COO_ITEMS;

// ---------------------------------------------------------------------------
// CSR/LibA/L — CSR-vector (kernels.py:167-189)
//
// Reference order: lane j%L of a row accumulates elements j, j+L, ...
// sequentially from 0, then the halving tree lanes[:h] += lanes[h:2h].
// A warp takes a tile of 32 rows and picks the effective lane count
// Lp = min(L, next_pow2(longest row in the tile)).  This is exact: lanes
// >= len only ever hold +0.0, so the tree steps h >= Lp each add +0.0 —
// the first turns a -0.0 partial into +0.0, the rest are no-ops — and the
// remaining steps are precisely the Lp-lane tree.  Short rows therefore get
// 32/Lp rows per warp instead of one, and U row groups are interleaved so
// every thread keeps U independent load chains in flight.
// ---------------------------------------------------------------------------
template <class T, class P, int L>
__global__ void __launch_bounds__(256) k_csr_vector(int64_t nrows, const P* __restrict__ ptr,
                                                    const int* __restrict__ cols,
                                                    const T* __restrict__ vals,
                                                    const T* __restrict__ x, T* __restrict__ y) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t0 = warp * 32; t0 < nrows; t0 += nwarps * 32) {   // warp-uniform
    const int64_t myrow = t0 + lane;
    int64_t ms = 0, ml = 0;
    if (myrow < nrows) {
      ms = ptr[myrow];
      ml = ptr[myrow + 1] - ms;
    }
    const unsigned longest = __reduce_max_sync(0xffffffffu, (unsigned)(ml < (1 << 30) ? ml : (1 << 30)));
    int Lp = 1;
    while (Lp < L && (unsigned)Lp < longest) Lp <<= 1;
    const int G = 32 / Lp;          // rows per group
    const int sub = lane & (Lp - 1);
    const int slot = lane / Lp;
    for (int g0 = 0; g0 < Lp; g0 += U) {   // Lp groups cover the 32-row tile
      int64_t s[U], len[U];
      T acc[U];
      int64_t most = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = (g0 + u) * G + slot;           // row within the tile
        const int src = q < 32 ? q : 0;
        s[u] = __shfl_sync(0xffffffffu, ms, src);
        len[u] = __shfl_sync(0xffffffffu, ml, src);
        if (g0 + u >= Lp || q >= 32) len[u] = 0;
        acc[u] = T(0);
        most = len[u] > most ? len[u] : most;
      }
      for (int64_t t = sub; t < most; t += Lp) {
        T v[U];
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (t < len[u]) {
            v[u] = ld_stream(vals + s[u] + t);
            c[u] = ld_stream(cols + s[u] + t);
          }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (t < len[u]) acc[u] = acc[u] + v[u] * ld_x(x + c[u]);
      }
      if (Lp < L) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = acc[u] + T(0);
      }
      for (int h = Lp >> 1; h >= 1; h >>= 1) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = acc[u] + __shfl_down_sync(0xffffffffu, acc[u], h, Lp);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = (g0 + u) * G + slot;
        if (sub == 0 && g0 + u < Lp && q < 32 && t0 + q < nrows) y[t0 + q] = acc[u];
      }
    }
  }
}
// ---------------------------------------------------------------------------
// CSR/LibB (row-scalar, kernels.py:192-199) and CSR/LibC (merge-path chunks,
// kernels.py:202-223): each CTA stages the products of its 128 rows into
// shared memory with coalesced loads, then every thread reduces its own row
// in the reference's reduceat order.  For LibC the row is cut at the chunk
// bounds and the pieces are added from 0 in chunk order.  CTAs whose rows
// exceed the staging capacity (long rows) read their products from global.
// ---------------------------------------------------------------------------
// CSR-vector order for one thread: the reference's L-lane halving tree
// (kernels.py:176-189) written as a recursion over lane subsets — the final
// value is tree(evens) + tree(odds), recursively, and leaf t is the
// sequential sum of elements t, t+L, ... .  Only Lp = min(L, next_pow2(len))
// lanes are materialised: the higher lanes only ever hold +0.0 and leaves
// are sums started from +0.0 (never -0.0), so the skipped tree steps are
// exact no-ops.
template <int LEVEL, class T, class G>
__device__ __forceinline__ T lane_tree(const G& get, int64_t s, int64_t len, int L, int t, int stride) {
  if constexpr (LEVEL == 0) {
    T leaf = T(0);
    for (int64_t k = t; k < len; k += L) leaf = leaf + get(s + k);
    return leaf;
  } else {
    const T even = lane_tree<LEVEL - 1, T>(get, s, len, L, t, 2 * stride);
    const T odd = lane_tree<LEVEL - 1, T>(get, s, len, L, t + stride, 2 * stride);
    return even + odd;
  }
}

template <class T, class G>
__device__ __forceinline__ T lane_tree_sum(const G& get, int64_t s, int64_t len, int L) {
  int bits = 0;
  while ((1 << bits) < L && (1 << bits) < len) ++bits;
  switch (bits) {
    case 0: return lane_tree<0, T>(get, s, len, L, 0, 1);
    case 1: return lane_tree<1, T>(get, s, len, L, 0, 1);
    case 2: return lane_tree<2, T>(get, s, len, L, 0, 1);
    case 3: return lane_tree<3, T>(get, s, len, L, 0, 1);
    case 4: return lane_tree<4, T>(get, s, len, L, 0, 1);
    default: return lane_tree<5, T>(get, s, len, L, 0, 1);
  }
}

template <class T, class P>
__device__ __forceinline__ T row_value(const T* sp, int64_t E0, bool staged, int64_t s, int64_t e,
                                       const int* __restrict__ cols, const T* __restrict__ vals,
                                       const T* __restrict__ x, const int64_t* __restrict__ bounds,
                                       int nb, int lanes) {
  auto get_s = [&](int64_t k) { return sp[k - E0]; };
  auto get_g = [&](int64_t k) { return ld_stream(vals + k) * ld_x(x + ld_stream(cols + k)); };
  if (lanes > 0) return staged ? lane_tree_sum<T>(get_s, s, e - s, lanes) : lane_tree_sum<T>(get_g, s, e - s, lanes);
  if (bounds == nullptr) {
    if (e == s) return T(0);
    return staged ? segment_sum<T>(get_s, s, e) : segment_sum<T>(get_g, s, e);
  }
  // LibC: first chunk bound strictly greater than s
  int lo = 0, hi = nb;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (bounds[mid] <= s) lo = mid + 1; else hi = mid;
  }
  T acc = T(0);
  int64_t cur = s;
  while (cur < e) {
    int64_t nxt = (lo < nb && bounds[lo] < e) ? bounds[lo] : e;
    T piece = staged ? segment_sum<T>(get_s, cur, nxt) : segment_sum<T>(get_g, cur, nxt);
    acc = acc + piece;
    cur = nxt;
    ++lo;
  }
  return acc;
}

template <class T, class P>
__global__ void __launch_bounds__(ROWSEG_ROWS) k_csr_rowseg(int64_t nrows, const P* __restrict__ ptr,
                                                            const int* __restrict__ cols,
                                                            const T* __restrict__ vals,
                                                            const T* __restrict__ x, T* __restrict__ y,
                                                            const int64_t* __restrict__ bounds, int nb,
                                                            int lanes) {
  __shared__ int64_t sptr[ROWSEG_ROWS + 1];
  __shared__ T sp[ROWSEG_CAP];
  const int64_t r0 = (int64_t)blockIdx.x * ROWSEG_ROWS;
  const int nr = (int)(nrows - r0 < ROWSEG_ROWS ? nrows - r0 : ROWSEG_ROWS);
  for (int i = threadIdx.x; i <= nr; i += blockDim.x) sptr[i] = ptr[r0 + i];
  __syncthreads();
  const int64_t E0 = sptr[0], E1 = sptr[nr];
  const bool staged = (E1 - E0) <= ROWSEG_CAP;
  if (staged) {
    constexpr int U = 4;
    for (int64_t k = E0 + threadIdx.x; k < E1; k += (int64_t)ROWSEG_ROWS * U) {
      T v[U];
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t kk = k + (int64_t)u * ROWSEG_ROWS;
        if (kk < E1) {
          v[u] = ld_stream(vals + kk);
          c[u] = ld_stream(cols + kk);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t kk = k + (int64_t)u * ROWSEG_ROWS;
        if (kk < E1) sp[kk - E0] = v[u] * ld_x(x + c[u]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < nr) {
    const int64_t s = sptr[threadIdx.x], e = sptr[threadIdx.x + 1];
    y[r0 + threadIdx.x] = row_value<T, P>(sp, E0, staged, s, e, cols, vals, x, bounds, nb, lanes);
  }
}

// ---------------------------------------------------------------------------
// COO/LibA (kernels.py:146-153) and the HYB spill (kernels.py:267-271):
// tile-per-CTA segmented reduction over row-sorted coordinates.  A segment
// (row run) belongs to the tile holding its head; runs crossing the tile end
// continue from global memory.  ADD accumulates into y (HYB), otherwise y
// must be zero-filled beforehand (rows without entries stay 0).
// ---------------------------------------------------------------------------
template <class T, bool ADD>
__global__ void __launch_bounds__(COO_THREADS) k_coo_segreduce(int64_t nnz,
                                                               const int* __restrict__ rows,
                                                               const int* __restrict__ cols,
                                                               const T* __restrict__ vals,
                                                               const T* __restrict__ x,
                                                               T* __restrict__ y) {
  __shared__ int srow[COO_TILE];
  __shared__ T sp[COO_TILE];
  const int64_t t0 = (int64_t)blockIdx.x * COO_TILE;
  const int n = (int)(nnz - t0 < COO_TILE ? nnz - t0 : COO_TILE);
  {
    T v[COO_ITEMS];
    int c[COO_ITEMS];
#pragma unroll
    for (int u = 0; u < COO_ITEMS; ++u) {
      const int k = threadIdx.x + u * COO_THREADS;
      if (k < n) {
        v[u] = ld_stream(vals + t0 + k);
        c[u] = ld_stream(cols + t0 + k);
        srow[k] = ld_stream(rows + t0 + k);
      }
    }
#pragma unroll
    for (int u = 0; u < COO_ITEMS; ++u) {
      const int k = threadIdx.x + u * COO_THREADS;
      if (k < n) sp[k] = v[u] * ld_x(x + c[u]);
    }
  }
  __syncthreads();
  const int64_t t1 = t0 + n;
  auto get = [&](int64_t g) {
    return g < t1 ? sp[g - t0] : ld_stream(vals + g) * ld_x(x + ld_stream(cols + g));
  };
  for (int k = threadIdx.x; k < n; k += COO_THREADS) {
    const int row = srow[k];
    const int prev = k > 0 ? srow[k - 1] : (t0 > 0 ? rows[t0 - 1] : -1);
    if (row == prev) continue;
    int e = k + 1;
    while (e < n && srow[e] == row) ++e;
    int64_t gend = t0 + e;
    if (e == n)
      while (gend < nnz && rows[gend] == row) ++gend;
    const T val = segment_sum<T>(get, t0 + k, gend);
    if (ADD) y[row] = y[row] + val;
    else y[row] = val;
  }
}

// ---------------------------------------------------------------------------
// COO/LibB (kernels.py:156-164): scatter-accumulate with fp64 atomics.  Runs
// of equal rows inside a warp are pre-summed with a segmented shuffle scan so
// only one atomic per run is issued.  Like the reference, the summation
// order is not deterministic (1e-8 equivalence bar, test_kernels.py:82).
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) k_coo_atomic(int64_t nnz, const int* __restrict__ rows,
                                                    const int* __restrict__ cols,
                                                    const T* __restrict__ vals,
                                                    const T* __restrict__ x, T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; base < nnz;
       base += stride) {
    const int64_t k = base + lane;
    int row = -1;
    T p = T(0);
    if (k < nnz) {
      row = ld_stream(rows + k);
      p = ld_stream(vals + k) * ld_x(x + ld_stream(cols + k));
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T o = __shfl_up_sync(0xffffffffu, p, d);
      const int orow = __shfl_up_sync(0xffffffffu, row, d);
      if (lane >= d && orow == row) p = p + o;
    }
    const int nrow = __shfl_down_sync(0xffffffffu, row, 1);
    if (row >= 0 && (lane == 31 || nrow != row)) atomicAdd(y + row, p);
  }
}

// ---------------------------------------------------------------------------
// ELL/LibA (kernels.py:226-233) and the HYB ELL part: thread per row, one
// coalesced column-major slice per stored column, sentinel -> exact +0.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) k_ell_sweep(int64_t nrows, int64_t ncols, int64_t width,
                                                   const int* __restrict__ cols,
                                                   const T* __restrict__ vals,
                                                   const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    T acc = T(0);
    int64_t k = 0;
    for (; k + 4 <= width; k += 4) {
      T v[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = ld_stream(cols + (k + u) * nrows + i);
        v[u] = ld_stream(vals + (k + u) * nrows + i);
        xv[u] = c < ncols ? ld_x(x + c) : T(0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = acc + v[u] * xv[u];
    }
    for (; k < width; ++k) {
      const int c = ld_stream(cols + k * nrows + i);
      const T v = ld_stream(vals + k * nrows + i);
      acc = acc + v * (c < ncols ? ld_x(x + c) : T(0));
    }
    y[i] = acc;
  }
}

// ELL/LibC (kernels.py:236-248): S = min(workers, width) strided partials per
// row, each summed from 0 over k = w, w+S, ..., merged into 0 in order w.
template <class T>
__global__ void __launch_bounds__(256) k_ell_strided(int64_t nrows, int64_t ncols, int64_t width,
                                                     int S, const int* __restrict__ cols,
                                                     const T* __restrict__ vals,
                                                     const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int w = 0; w < S; ++w) {
      T part = T(0);
      for (int64_t k = w; k < width; k += S) {
        const int c = ld_stream(cols + k * nrows + i);
        const T v = ld_stream(vals + k * nrows + i);
        part = part + v * (c < ncols ? ld_x(x + c) : T(0));
      }
      acc = acc + part;
    }
    y[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// DIA/LibA (kernels.py:251-260): thread per row, ascending offsets, cells
// whose column leaves the matrix are skipped (not added).
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) k_dia(int64_t nrows, int64_t ncols, int64_t ndiag,
                                             const long long* __restrict__ offs,
                                             const T* __restrict__ data, const T* __restrict__ x,
                                             T* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    T acc = T(0);
    int64_t k = 0;
    for (; k + 4 <= ndiag; k += 4) {
      T v[4], xv[4];
      bool in[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + __ldg(offs + k + u);
        in[u] = j >= 0 && j < ncols;
        v[u] = ld_stream(data + (k + u) * nrows + i);
        xv[u] = in[u] ? ld_x(x + j) : T(0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (in[u]) acc = acc + v[u] * xv[u];
    }
    for (; k < ndiag; ++k) {
      const int64_t j = i + __ldg(offs + k);
      if (j >= 0 && j < ncols) acc = acc + ld_stream(data + k * nrows + i) * ld_x(x + j);
    }
    y[i] = acc;
  }
}

// spmv_reference (formats.py:419-435): strictly sequential row sums from 0.
template <class P>
__global__ void __launch_bounds__(256) k_csr_sequential(int64_t nrows, const P* __restrict__ ptr,
                                                        const int* __restrict__ cols,
                                                        const double* __restrict__ vals,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) acc = acc + vals[k] * __ldg(x + cols[k]);
    y[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
static bool supported(int fmt, int lib) {
  // SUPPORT_TABLE (kernels.py:43-47)
  if (lib == SVB_LIBA) return fmt >= SVB_COO && fmt <= SVB_HYB;
  if (lib == SVB_LIBB) return fmt == SVB_COO || fmt == SVB_CSR;
  if (lib == SVB_LIBC) return fmt == SVB_CSR || fmt == SVB_ELL;
  return false;
}

static const char* fmt_name(int f) {
  static const char* names[] = {"COO", "CSR", "ELL", "DIA", "HYB"};
  return (f >= 0 && f <= 4) ? names[f] : "?";
}

// LibC chunk edges: np.linspace(0, nnz, min(workers, nnz) + 1, dtype=int64)
// (kernels.py:209-210).  numpy computes i*step in float64 (step = nnz/chunks),
// floors for integer dtypes and pins the last edge to nnz.
std::vector<int64_t> merge_bounds(int64_t nnz, int64_t workers) {
  const int64_t chunks = std::min<int64_t>(workers, nnz);
  std::vector<int64_t> b(chunks + 1);
  const double step = (double)nnz / (double)chunks;
  for (int64_t c = 0; c < chunks; ++c) b[c] = (int64_t)std::floor((double)c * step);
  b[chunks] = nnz;
  return b;
}

struct BoundsCache {
  std::mutex mu;
  std::map<std::pair<const svb_matrix*, int64_t>, Buf> map;
};
static BoundsCache& bounds_cache() {
  static BoundsCache c;
  return c;
}

// Device copy of the LibC bounds for (matrix, workers).  Cached per handle:
// the solver calls the same configuration every iteration.
static const int64_t* device_bounds(const svb_matrix* m, int64_t workers, int* nb, cudaStream_t s) {
  std::vector<int64_t> h = merge_bounds(m->nnz, workers);
  *nb = (int)h.size();
  auto& c = bounds_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto key = std::make_pair(m, workers);
  auto it = c.map.find(key);
  if (it != c.map.end() && it->second->bytes == h.size() * 8) return ptr<int64_t>(it->second);
  Buf b = alloc(h.size() * 8, s);
  SVB_CUDA_TRY(cudaMemcpyAsync(b->ptr, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s));
  SVB_CUDA_TRY(cudaStreamSynchronize(s));  // h is a host temporary
  detach(b);
  c.map[key] = b;
  return ptr<int64_t>(b);
}

void forget_bounds(const svb_matrix* m) {
  auto& c = bounds_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  for (auto it = c.map.begin(); it != c.map.end();)
    it = (it->first.first == m) ? c.map.erase(it) : std::next(it);
}

constexpr int64_t LANE_STAGED_MAX_ROW = 64;

__global__ void k_row_max(int64_t nrows, const int* __restrict__ p32, const long long* __restrict__ p64,
                          unsigned long long* out) {
  int64_t best = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = p64 ? p64[i + 1] - p64[i] : (int64_t)p32[i + 1] - p32[i];
    best = len > best ? len : best;
  }
  for (int o = 16; o; o >>= 1) {
    const int64_t other = __shfl_xor_sync(0xffffffffu, (long long)best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)best);
}

// Longest row of a CSR handle, computed once and cached on the handle.
static int64_t csr_max_row_len(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->max_row_len < 0) {
    Buf d = alloc(8, s);
    SVB_CUDA_TRY(cudaMemsetAsync(d->ptr, 0, 8, s));
    k_row_max<<<grid_for(m->nrows, 256), 256, 0, s>>>(m->nrows, m->ptr64 ? nullptr : ptr<int>(m->ptr),
                                                      m->ptr64 ? ptr<long long>(m->ptr) : nullptr,
                                                      ptr<unsigned long long>(d));
    SVB_CHECK_LAUNCH();
    unsigned long long h = 0;
    SVB_CUDA_TRY(cudaMemcpyAsync(&h, d->ptr, 8, cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    m->max_row_len = (int64_t)h;
  }
  return m->max_row_len;
}

template <class T>
static void launch_spmv(const svb_matrix* m, int fmt, int lib, int lane, int workers,
                        const T* vals, const T* svals, const T* x, T* y, cudaStream_t s) {
  const int64_t n = m->nrows;
  if (fmt == SVB_CSR) {
    if (lib == SVB_LIBA && !(lane == 2 || lane == 4 || lane == 8 || lane == 16 || lane == 32))
      throw Error{SVB_UNSUPPORTED_CONFIG, "lane_width must be one of (2, 4, 8, 16, 32)"};
    if (lib == SVB_LIBA && csr_max_row_len(m, s) > LANE_STAGED_MAX_ROW) {
      // long rows: the warp kernel keeps L lanes per row busy
      const unsigned g = grid_for(n * lane, 256, 8);
#define SVB_VEC(LL)                                                                        \
  case LL:                                                                                 \
    if (m->ptr64)                                                                          \
      k_csr_vector<T, long long, LL><<<g, 256, 0, s>>>(n, ptr<long long>(m->ptr),          \
                                                       ptr<int>(m->cols), vals, x, y);     \
    else                                                                                   \
      k_csr_vector<T, int, LL><<<g, 256, 0, s>>>(n, ptr<int>(m->ptr), ptr<int>(m->cols),   \
                                                 vals, x, y);                              \
    break;
      switch (lane) {
        SVB_VEC(2)
        SVB_VEC(4)
        SVB_VEC(8)
        SVB_VEC(16)
        SVB_VEC(32)
      }
#undef SVB_VEC
    } else {
      // short rows (and LibB / LibC): CTA-staged rows, one thread per row,
      // reduced in the configuration's exact order
      const int64_t* bounds = nullptr;
      int nb = 0;
      const int lanes = lib == SVB_LIBA ? lane : 0;
      if (lib == SVB_LIBC) {
        if (m->nnz == 0) {
          SVB_CUDA_TRY(cudaMemsetAsync(y, 0, n * sizeof(T), s));
          return;
        }
        bounds = device_bounds(m, workers, &nb, s);
      }
      const unsigned g = (unsigned)((n + ROWSEG_ROWS - 1) / ROWSEG_ROWS);
      if (m->ptr64)
        k_csr_rowseg<T, long long><<<g, ROWSEG_ROWS, 0, s>>>(n, ptr<long long>(m->ptr), ptr<int>(m->cols),
                                                             vals, x, y, bounds, nb, lanes);
      else
        k_csr_rowseg<T, int><<<g, ROWSEG_ROWS, 0, s>>>(n, ptr<int>(m->ptr), ptr<int>(m->cols), vals, x, y,
                                                       bounds, nb, lanes);
    }
  } else if (fmt == SVB_COO) {
    SVB_CUDA_TRY(cudaMemsetAsync(y, 0, n * sizeof(T), s));
    if (m->nnz == 0) return;
    if (lib == SVB_LIBA) {
      const unsigned g = (unsigned)((m->nnz + COO_TILE - 1) / COO_TILE);
      k_coo_segreduce<T, false><<<g, COO_THREADS, 0, s>>>(m->nnz, ptr<int>(m->rows), ptr<int>(m->cols),
                                                          vals, x, y);
    } else {
      k_coo_atomic<T><<<grid_for(m->nnz, 256, 16), 256, 0, s>>>(m->nnz, ptr<int>(m->rows),
                                                               ptr<int>(m->cols), vals, x, y);
    }
  } else if (fmt == SVB_ELL) {
    if (lib == SVB_LIBA || m->width == 0)
      k_ell_sweep<T><<<grid_for(n, 256, 8), 256, 0, s>>>(n, m->ncols, m->width, ptr<int>(m->cols), vals, x, y);
    else {
      const int S = (int)std::min<int64_t>(workers, m->width);
      k_ell_strided<T><<<grid_for(n, 256, 8), 256, 0, s>>>(n, m->ncols, m->width, S, ptr<int>(m->cols),
                                                           vals, x, y);
    }
  } else if (fmt == SVB_DIA) {
    k_dia<T><<<grid_for(n, 256, 8), 256, 0, s>>>(n, m->ncols, m->ndiag, ptr<long long>(m->offs), vals, x, y);
  } else {  // HYB
    k_ell_sweep<T><<<grid_for(n, 256, 8), 256, 0, s>>>(n, m->ncols, m->width, ptr<int>(m->cols), vals, x, y);
    if (m->spill_nnz > 0) {
      SVB_CHECK_LAUNCH();
      const unsigned g = (unsigned)((m->spill_nnz + COO_TILE - 1) / COO_TILE);
      k_coo_segreduce<T, true><<<g, COO_THREADS, 0, s>>>(m->spill_nnz, ptr<int>(m->rows),
                                                         ptr<int>(m->scols), svals, x, y);
    }
  }
  SVB_CHECK_LAUNCH();
}

void spmv_dispatch(const svb_matrix* m, int fmt, int lib, int lane, int workers, int dtype,
                   const void* x, void* y, cudaStream_t s) {
  SVB_REQUIRE(m, SVB_INVALID, "null matrix handle");
  SVB_REQUIRE(supported(fmt, lib), SVB_UNSUPPORTED_CONFIG, "configuration not in the support table");
  if (m->fmt != fmt)
    throw Error{SVB_UNSUPPORTED_CONFIG, std::string("matrix is stored as ") + fmt_name(m->fmt) +
                                            ", kernel expects " + fmt_name(fmt)};
  SVB_REQUIRE(workers >= 1, SVB_INVALID, "workers must be >= 1");
  if (m->nrows == 0) return;
  if (dtype == SVB_F64) {
    launch_spmv<double>(m, fmt, lib, lane, workers, ptr<double>(m->vals), ptr<double>(m->svals),
                        static_cast<const double*>(x), static_cast<double*>(y), s);
  } else if (dtype == SVB_F32) {
    const float* v = vals_f32(m, s);
    const float* sv = (fmt == SVB_HYB) ? svals_f32(m, s) : nullptr;
    launch_spmv<float>(m, fmt, lib, lane, workers, v, sv, static_cast<const float*>(x),
                       static_cast<float*>(y), s);
  } else {
    throw Error{SVB_INVALID, "dtype must be SVB_F64 or SVB_F32"};
  }
}

}  // namespace svb

using namespace svb;

extern "C" {

int svb_spmv(const svb_matrix* m, int format, int library, int lane, int workers, int dtype,
             const void* x_dev, void* y_dev, void* stream) {
  return guard([&] {
    spmv_dispatch(m, format, library, lane, workers, dtype, x_dev, y_dev,
                  reinterpret_cast<cudaStream_t>(stream));
  });
}

int svb_spmv_host(const svb_matrix* m, int format, int library, int lane, int workers,
                  const double* x_host, double* y_host, void* stream) {
  return guard([&] {
    SVB_REQUIRE(m, SVB_INVALID, "null matrix handle");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Buf x = upload(x_host, m->ncols * 8, s);
    Buf y = alloc(m->nrows * 8, s);
    spmv_dispatch(m, format, library, lane, workers, SVB_F64, x->ptr, y->ptr, s);
    SVB_CUDA_TRY(cudaMemcpyAsync(y_host, y->ptr, m->nrows * 8, cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
  });
}

int svb_spmv_sequential(const svb_matrix* m, const double* x_dev, double* y_dev, void* stream) {
  return guard([&] {
    SVB_REQUIRE(m && m->fmt == SVB_CSR, SVB_UNSUPPORTED_CONFIG, "spmv_sequential expects CSR");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (m->ptr64)
      k_csr_sequential<long long><<<grid_for(m->nrows, 256), 256, 0, s>>>(
          m->nrows, ptr<long long>(m->ptr), ptr<int>(m->cols), ptr<double>(m->vals), x_dev, y_dev);
    else
      k_csr_sequential<int><<<grid_for(m->nrows, 256), 256, 0, s>>>(
          m->nrows, ptr<int>(m->ptr), ptr<int>(m->cols), ptr<double>(m->vals), x_dev, y_dev);
    SVB_CHECK_LAUNCH();
  });
}

}  // extern "C"
