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
//   COO/LibA     reduceat over row runs                    -> row kernel on cached run starts
//   COO/LibB     np.add.at, random order                   -> warp-aggregated atomics
//   ELL/LibA     column sweep from 0                       -> thread per row
//   ELL/LibC     S strided partials, merged in order       -> thread per row
//   DIA/LibA     ascending-offset sweep                    -> thread per row
//   HYB/LibA     ELL sweep, then += reduceat(spill runs)   -> ELL + row kernel (add)
// All kernels are bandwidth-bound (~2 flop per 12-16 B): no tensor cores.
#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "matrix.cuh"

namespace svb {

constexpr int ROWSEG_ROWS = 128;     // rows per CTA of the staged row-segment kernel
constexpr int ROWSEG_CAP = 2048;     // staged products per CTA

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

// ---------------------------------------------------------------------------
// Helpers shared by the exact row reductions
// ---------------------------------------------------------------------------
constexpr int LONG_ROW = 128;    // pairwise rows longer than this are reduced by a whole warp
constexpr int LONG_LANE_ROW = 32;  // lane-tree rows longer than this likewise (L lanes, coalesced)
constexpr int WARP_LEAVES = 64;  // leaf slots per warp for long pairwise segments

// LibB: p[s] + pairwise(p[s+1:e]); LibC: the row cut at the chunk bounds,
// each piece reduced that way and added from 0 in chunk order.
template <class T, class G>
__device__ __forceinline__ T pw_row_value(const G& get, int64_t s, int64_t e, const int64_t* __restrict__ bounds,
                                          int nb) {
  if (bounds == nullptr) return e == s ? T(0) : segment_sum<T>(get, s, e);
  int lo = 0, hi = nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (bounds[mid] <= s) lo = mid + 1; else hi = mid;
  }
  T acc = T(0);
  for (int64_t cur = s; cur < e; ++lo) {
    const int64_t nxt = (lo < nb && bounds[lo] < e) ? bounds[lo] : e;
    acc = acc + segment_sum<T>(get, cur, nxt);
    cur = nxt;
  }
  return acc;
}

// Warp-cooperative p[s] + pairwise(p[s+1:e]) for one long segment: lane 0
// enumerates the recursion's leaves, 8 lanes evaluate each leaf (one lane
// per numpy accumulator, combined with the same ((r0+r1)+(r2+r3))+... tree),
// then lane 0 combines the leaf sums along the recursion.  Result on lane 0.
template <class T, class G>
__device__ T warp_pw_segment(const G& get, int64_t s, int64_t e, int64_t* loff, int* llen, T* lsum) {
  const int lane = threadIdx.x & 31;
  const int64_t m = e - s - 1;  // elements of the pairwise part
  if (m <= 0) return get(s);
  int nleaf = 0;
  if (lane == 0) {
    pw_traverse<T>([&](int64_t lo, int64_t n) {
      if (nleaf < WARP_LEAVES) {
        loff[nleaf] = lo;
        llen[nleaf] = (int)n;
      }
      ++nleaf;
      return T(0);
    }, s + 1, m);
  }
  nleaf = __shfl_sync(0xffffffffu, nleaf, 0);
  if (nleaf > WARP_LEAVES) {  // extremely long segment: sequential fallback
    T r = T(0);
    if (lane == 0) r = segment_sum<T>(get, s, e);
    return r;
  }
  __syncwarp();
  const int grp = lane >> 3, k = lane & 7;
  for (int l0 = 0; l0 < nleaf; l0 += 4) {
    const int li = l0 + grp;
    T r = T(0);
    int64_t lo = 0;
    int n = 0;
    if (li < nleaf) {
      lo = loff[li];
      n = llen[li];
    }
    if (n >= 8) {
      r = get(lo + k);
      const int lim = n - (n % 8);
      for (int i = 8; i < lim; i += 8) r = r + get(lo + i + k);
    }
    // fixed combine tree inside each 8-lane group
    T o = __shfl_down_sync(0xffffffffu, r, 1);
    if ((k & 1) == 0) r = r + o;
    o = __shfl_down_sync(0xffffffffu, r, 2);
    if ((k & 3) == 0) r = r + o;
    o = __shfl_down_sync(0xffffffffu, r, 4);
    if (k == 0) r = r + o;
    if (k == 0 && li < nleaf) {
      if (n < 8) {
        T q = T(-0.0);
        for (int i = 0; i < n; ++i) q = q + get(lo + i);
        r = q;
      } else {
        for (int i = n - (n % 8); i < n; ++i) r = r + get(lo + i);
      }
      lsum[li] = r;
    }
  }
  __syncwarp();
  T total = T(0);
  if (lane == 0) {
    int next = 0;
    total = pw_traverse<T>([&](int64_t, int64_t) { return lsum[next++]; }, s + 1, m);
    total = get(s) + total;
  }
  return total;
}

// Warp-cooperative L-lane CSR-vector row (len > LONG_ROW >= L): lane t < L
// sums elements t, t+L, ... in order; halving tree.  Result on lane 0.
template <class T, class G>
__device__ T warp_lane_row(const G& get, int64_t s, int64_t len, int L) {
  const int lane = threadIdx.x & 31;
  T acc = T(0);
  if (lane < L)
    for (int64_t k = lane; k < len; k += L) acc = acc + get(s + k);
  for (int h = L >> 1; h >= 1; h >>= 1) {
    const T o = __shfl_down_sync(0xffffffffu, acc, h);
    if (lane < h) acc = acc + o;
  }
  return acc;
}

// ---------------------------------------------------------------------------
// CSR/LibA/L (kernels.py:167-189), CSR/LibB (kernels.py:192-199) and
// CSR/LibC (kernels.py:202-223).  Each CTA owns 128 consecutive rows; all
// threads stage the rows' products p = v*x[c] in shared memory with
// coalesced loads and U independent gathers in flight per thread; then one
// thread per row reduces it in the configuration's exact order (lane tree,
// numpy pairwise, or chunk pieces) and rows longer than LONG_ROW are reduced
// by a whole warp (leaf-parallel pairwise / L lanes).  CTAs whose entries
// exceed the staging capacity read their products from global memory.
// ---------------------------------------------------------------------------
template <class T, class P, bool ADD>
__global__ void __launch_bounds__(ROWSEG_ROWS) k_csr_rowseg(int64_t nrows, const P* __restrict__ ptr,
                                                            const int* __restrict__ cols,
                                                            const T* __restrict__ vals,
                                                            const T* __restrict__ x, T* __restrict__ y,
                                                            const int64_t* __restrict__ bounds, int nb,
                                                            int lanes) {
  __shared__ int64_t sptr[ROWSEG_ROWS + 1];
  __shared__ T sp[ROWSEG_CAP];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * ROWSEG_ROWS;
  const int nr = (int)(nrows - r0 < ROWSEG_ROWS ? nrows - r0 : ROWSEG_ROWS);
  for (int i = tid; i <= nr; i += blockDim.x) sptr[i] = ptr[r0 + i];
  __syncthreads();
  const int64_t E0 = sptr[0];
  // stage the CTA's products (a prefix when long rows push it past capacity)
  const int64_t E1 = sptr[nr] - E0 <= ROWSEG_CAP ? sptr[nr] : E0 + ROWSEG_CAP;
  {
    constexpr int U = 4;
    for (int64_t k = E0 + tid; k < E1; k += (int64_t)ROWSEG_ROWS * U) {
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
  auto get_s = [&](int64_t k) { return sp[k - E0]; };
  auto get_g = [&](int64_t k) { return ld_stream(vals + k) * ld_x(x + ld_stream(cols + k)); };
  if (tid < nr) {
    const int64_t s = sptr[tid], e = sptr[tid + 1];
    if (e - s <= (lanes > 0 ? LONG_LANE_ROW : LONG_ROW)) {
      const bool staged = e <= E1;
      T v;
      if (lanes > 0) v = staged ? lane_tree_sum<T>(get_s, s, e - s, lanes) : lane_tree_sum<T>(get_g, s, e - s, lanes);
      else v = staged ? pw_row_value<T>(get_s, s, e, bounds, nb) : pw_row_value<T>(get_g, s, e, bounds, nb);
      if (!ADD) y[r0 + tid] = v;
      else if (e > s) y[r0 + tid] = y[r0 + tid] + v;   // HYB spill: rows with entries only
    }
  }
  // rows longer than LONG_ROW are reduced by k_long_rows
}
// ---------------------------------------------------------------------------
// Long rows / runs (> LONG_ROW entries) of any row-sorted layout: one warp
// per segment from a per-handle list, so the few heavy rows of a power-law
// matrix run side by side instead of serialising inside one CTA.  Exact
// order as the thread path (lane tree / pairwise / chunk pieces).
// ---------------------------------------------------------------------------
template <class T, bool ADD>
__global__ void __launch_bounds__(128) k_long_rows(int64_t nlong, const int* __restrict__ lrow,
                                                   const int64_t* __restrict__ lbeg, const int64_t* __restrict__ lend,
                                                   const int* __restrict__ cols, const T* __restrict__ vals,
                                                   const T* __restrict__ x, T* __restrict__ y,
                                                   const int64_t* __restrict__ bounds, int nb, int lanes) {
  __shared__ int64_t loff[4][WARP_LEAVES];
  __shared__ int llen[4][WARP_LEAVES];
  __shared__ T lsum[4][WARP_LEAVES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto get = [&](int64_t k) { return ld_stream(vals + k) * ld_x(x + ld_stream(cols + k)); };
  for (int64_t i = (int64_t)blockIdx.x * 4 + warp; i < nlong; i += (int64_t)gridDim.x * 4) {
    const int64_t s = lbeg[i], e = lend[i];
    if (lanes == 0 && e - s <= LONG_ROW) continue;   // done by the thread path
    T v;
    if (lanes > 0) {
      v = warp_lane_row<T>(get, s, e - s, lanes);
    } else if (bounds == nullptr) {
      v = warp_pw_segment<T>(get, s, e, loff[warp], llen[warp], lsum[warp]);
    } else {
      int lo = 0, hi = nb;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (bounds[mid] <= s) lo = mid + 1; else hi = mid;
      }
      T acc = T(0);
      for (int64_t cur = s; cur < e; ++lo) {
        const int64_t nxt = (lo < nb && bounds[lo] < e) ? bounds[lo] : e;
        const T piece = warp_pw_segment<T>(get, cur, nxt, loff[warp], llen[warp], lsum[warp]);
        acc = acc + piece;
        cur = nxt;
      }
      v = acc;
    }
    if (lane == 0) {
      if (ADD) y[lrow[i]] = y[lrow[i]] + v;
      else y[lrow[i]] = v;
    }
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

// COO run starts as an int64 row pointer, derived once per handle
static const long long* coo_runs(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (!m->dptr) {
    m->dptr = rows_to_ptr(ptr<int32_t>(m->rows), m->nnz, m->nrows, true, s);
    detach(m->dptr);
  }
  return ptr<long long>(m->dptr);
}

// rows of a row pointer longer than LONG_LANE_ROW -> (row, begin, end) list
template <class P>
__global__ void k_find_long(int64_t nrows, const P* __restrict__ ptr, unsigned long long* count, int* lrow,
                            int64_t* lbeg, int64_t* lend) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = ptr[i], e = ptr[i + 1];
    if (e - b > LONG_LANE_ROW) {
      const unsigned long long k = atomicAdd(count, 1ull);
      lrow[k] = (int)i;
      lbeg[k] = b;
      lend[k] = e;
    }
  }
}

// The handle's long-segment list (built once, cached): CSR rows, COO runs
// (via a derived row pointer) or the HYB spill runs.
static int64_t long_list(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->nlong >= 0) return m->nlong;
  const int64_t entries = m->fmt == SVB_HYB ? m->spill_nnz : m->nnz;
  const int64_t cap = entries / (LONG_LANE_ROW + 1) + 1;
  m->lrow = alloc(cap * 4, s);
  m->lbeg = alloc(cap * 8, s);
  m->lend = alloc(cap * 8, s);
  detach(m->lrow);
  detach(m->lbeg);
  detach(m->lend);
  Buf cnt = alloc(8, s);
  SVB_CUDA_TRY(cudaMemsetAsync(cnt->ptr, 0, 8, s));
  const unsigned g = grid_for(m->nrows, 256);
  auto run = [&](auto* p) {
    k_find_long<<<g, 256, 0, s>>>(m->nrows, p, ptr<unsigned long long>(cnt), ptr<int>(m->lrow),
                                  ptr<int64_t>(m->lbeg), ptr<int64_t>(m->lend));
    SVB_CHECK_LAUNCH();
  };
  if (m->fmt == SVB_CSR) {
    if (m->ptr64) run(ptr<long long>(m->ptr));
    else run(ptr<int>(m->ptr));
  } else if (m->fmt == SVB_COO) {
    run(ptr<long long>(m->dptr));
  } else {  // HYB: spill row pointer (int64)
    run(ptr<long long>(m->ptr));
  }
  unsigned long long h = 0;
  SVB_CUDA_TRY(cudaMemcpyAsync(&h, cnt->ptr, 8, cudaMemcpyDeviceToHost, s));
  SVB_CUDA_TRY(cudaStreamSynchronize(s));
  m->nlong = (int64_t)h;
  return m->nlong;
}

template <class T, bool ADD>
static void launch_long(const svb_matrix* m, const int* cols, const T* vals, const T* x, T* y,
                        const int64_t* bounds, int nb, int lanes, cudaStream_t s) {
  const int64_t nl = long_list(m, s);
  if (nl <= 0) return;
  const unsigned g = (unsigned)((nl + 3) / 4);
  k_long_rows<T, ADD><<<g, 128, 0, s>>>(nl, ptr<int>(m->lrow), ptr<int64_t>(m->lbeg), ptr<int64_t>(m->lend),
                                        cols, vals, x, y, bounds, nb, lanes);
  SVB_CHECK_LAUNCH();
}

template <class T>
static void launch_spmv(const svb_matrix* m, int fmt, int lib, int lane, int workers,
                        const T* vals, const T* svals, const T* x, T* y, cudaStream_t s) {
  const int64_t n = m->nrows;
  if (fmt == SVB_CSR) {
    if (lib == SVB_LIBA && !(lane == 2 || lane == 4 || lane == 8 || lane == 16 || lane == 32))
      throw Error{SVB_UNSUPPORTED_CONFIG, "lane_width must be one of (2, 4, 8, 16, 32)"};
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
      k_csr_rowseg<T, long long, false><<<g, ROWSEG_ROWS, 0, s>>>(n, ptr<long long>(m->ptr), ptr<int>(m->cols),
                                                                  vals, x, y, bounds, nb, lanes);
    else
      k_csr_rowseg<T, int, false><<<g, ROWSEG_ROWS, 0, s>>>(n, ptr<int>(m->ptr), ptr<int>(m->cols), vals, x, y,
                                                            bounds, nb, lanes);
    SVB_CUDA_TRY(cudaGetLastError());   // counted by the final check below
    launch_long<T, false>(m, ptr<int>(m->cols), vals, x, y, bounds, nb, lanes, s);
  } else if (fmt == SVB_COO) {
    if (lib == SVB_LIBA) {
      // row runs of the sorted coordinates (kernels.py:141-153), reduced in
      // reduceat order by the row kernel; rows without entries get 0
      const long long* runs = coo_runs(m, s);
      const unsigned g = (unsigned)((n + ROWSEG_ROWS - 1) / ROWSEG_ROWS);
      k_csr_rowseg<T, long long, false><<<g, ROWSEG_ROWS, 0, s>>>(n, runs, ptr<int>(m->cols), vals, x, y,
                                                                  nullptr, 0, 0);
      SVB_CUDA_TRY(cudaGetLastError());
      launch_long<T, false>(m, ptr<int>(m->cols), vals, x, y, nullptr, 0, 0, s);
    } else {
      SVB_CUDA_TRY(cudaMemsetAsync(y, 0, n * sizeof(T), s));
      if (m->nnz == 0) return;
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
      const unsigned g = (unsigned)((n + ROWSEG_ROWS - 1) / ROWSEG_ROWS);
      k_csr_rowseg<T, long long, true><<<g, ROWSEG_ROWS, 0, s>>>(n, ptr<long long>(m->ptr), ptr<int>(m->scols),
                                                                 svals, x, y, nullptr, 0, 0);
      SVB_CUDA_TRY(cudaGetLastError());
      launch_long<T, true>(m, ptr<int>(m->scols), svals, x, y, nullptr, 0, 0, s);
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
