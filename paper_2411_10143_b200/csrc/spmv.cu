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
#include <cstdlib>
#include <type_traits>
#include <map>
#include <mutex>
#include <vector>

#include "matrix.cuh"

namespace svb {

constexpr int ROWSEG_ROWS = 128;     // threads of the row kernel = max rows per tile

// CSR-vector order for one thread: the reference's L-lane halving tree
// (kernels.py:176-189).  Leaf t is the sequential sum (from +0.0) of
// elements t, t+L, ...; the halving tree over the leaves equals a balanced
// binary tree over the leaves in bit-reversed order, evaluated here as a
// binary counter over compile-time leaf indices (registers only).  LP leaves
// are materialised, LP a power of two with min(L, next_pow2(len)) <= LP <= L:
// the skipped leaves are empty sums (+0.0) and no partial sum is ever -0.0,
// so the skipped tree steps are exact no-ops.
__host__ __device__ constexpr int bit_reverse(int r, int nbits) {
  int t = 0;
  for (int b = 0; b < nbits; ++b) t |= ((r >> b) & 1) << (nbits - 1 - b);
  return t;
}
__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

template <int LP, class T, class G>
__device__ __forceinline__ T lane_tree_fixed(const G& get, int len, int L) {
  constexpr int LOG = ilog2(LP);
  T lvl[LOG + 1];
#pragma unroll
  for (int r = 0; r < LP; ++r) {
    const int t = bit_reverse(r, LOG);
    T cur = T(0);
    for (int k = t; k < len; k += L) cur = cur + get(k);
    int level = 0;
#pragma unroll
    for (int b = 0; b < LOG; ++b) {
      if (((r + 1) >> b) & 1) break;
      cur = lvl[b] + cur;
      level = b + 1;
    }
    lvl[level] = cur;
  }
  return lvl[LOG];
}

// Warp-uniform dispatch: LP = min(L, next_pow2(longest row of the warp)).
template <class T, class G>
__device__ __forceinline__ T lane_tree_warp(const G& get, int len, int L, int warp_max_len) {
  int lp = 1;
  while (lp < L && lp < warp_max_len) lp <<= 1;
  switch (lp) {
    case 1: return lane_tree_fixed<1, T>(get, len, L);
    case 2: return lane_tree_fixed<2, T>(get, len, L);
    case 4: return lane_tree_fixed<4, T>(get, len, L);
    case 8: return lane_tree_fixed<8, T>(get, len, L);
    case 16: return lane_tree_fixed<16, T>(get, len, L);
    default: return lane_tree_fixed<32, T>(get, len, L);
  }
}

// ---------------------------------------------------------------------------
// Helpers shared by the exact row reductions
// ---------------------------------------------------------------------------
constexpr int THREAD_LANE_ROW = 32;   // lane-tree rows up to this: one thread per row
constexpr int THREAD_PW_ROW = 128;    // pairwise rows up to this: one thread per row
constexpr int MED_ROW = 1024;         // longer rows of a tile: one warp per row, from shared
                                      // memory (rows above MED_ROW: one CTA each, cta_long_row)
constexpr int MED_LEAVES = 16;        // pairwise leaves of a <= 1024-entry segment (max 9)

// LibB: p[s] + pairwise(p[s+1:e]); LibC: the row cut at the chunk bounds,
// each piece reduced that way and added from 0 in chunk order.
__device__ __forceinline__ int first_bound_after(const int64_t* __restrict__ bounds, int nb, int64_t s) {
  int lo = 0, hi = nb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (bounds[mid] <= s) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <class T, class G>
__device__ __forceinline__ T pw_row_value(const G& get, int64_t s, int64_t e, const int64_t* __restrict__ bounds,
                                          int nb) {
  if (bounds == nullptr) return e == s ? T(0) : segment_sum<T>(get, s, e);
  T acc = T(0);
  for (int64_t cur = s, lo = first_bound_after(bounds, nb, s); cur < e; ++lo) {
    const int64_t nxt = (lo < nb && bounds[lo] < e) ? bounds[lo] : e;
    acc = acc + segment_sum<T>(get, cur, nxt);
    cur = nxt;
  }
  return acc;
}

// Warp-cooperative pairwise(p[lo : lo+n]) for a subtree of at most CAP
// leaves: lane 0 enumerates the recursion's leaves, 8 lanes evaluate each
// leaf (one lane per numpy accumulator, combined with the same
// ((r0+r1)+(r2+r3))+... tree), then lane 0 combines the leaf sums along the
// recursion.  Called by the whole (converged) warp; result on every lane.
template <int CAP, class T, class G>
__device__ T warp_pw_block(const G& get, int64_t lo, int64_t n, int64_t* loff, int* llen, T* lsum) {
  const int lane = threadIdx.x & 31;
  int nleaf = 0;
  if (lane == 0) {
    pw_traverse<T>([&](int64_t l, int64_t m) {
      if (nleaf < CAP) {
        loff[nleaf] = l;
        llen[nleaf] = (int)m;
      }
      ++nleaf;
      return T(0);
    }, lo, n);
  }
  nleaf = __shfl_sync(0xffffffffu, nleaf, 0);
  __syncwarp();
  const int grp = lane >> 3, k = lane & 7;
  for (int l0 = 0; l0 < nleaf; l0 += 4) {
    const int li = l0 + grp;
    T r = T(0);
    int64_t b = 0;
    int m = 0;
    if (li < nleaf) {
      b = loff[li];
      m = llen[li];
    }
    if (m >= 8) {
      r = get(b + k);
      const int lim = m - (m % 8);
#pragma unroll 4
      for (int i = 8; i < lim; i += 8) r = r + get(b + i + k);
    }
    T o = __shfl_down_sync(0xffffffffu, r, 1);
    if ((k & 1) == 0) r = r + o;
    o = __shfl_down_sync(0xffffffffu, r, 2);
    if ((k & 3) == 0) r = r + o;
    o = __shfl_down_sync(0xffffffffu, r, 4);
    if (k == 0) r = r + o;
    if (k == 0 && li < nleaf) {
      if (m < 8) {
        T q = T(-0.0);
        for (int i = 0; i < m; ++i) q = q + get(b + i);
        r = q;
      } else {
        for (int i = m - (m % 8); i < m; ++i) r = r + get(b + i);
      }
      lsum[li] = r;
    }
  }
  __syncwarp();
  T total = T(0);
  if (lane == 0) {
    int next = 0;
    total = pw_traverse<T>([&](int64_t, int64_t) { return lsum[next++]; }, lo, n);
  }
  total = __shfl_sync(0xffffffffu, total, 0);
  __syncwarp();  // the leaf slots are reused by the next call
  return total;
}

// p[s] + pairwise(p[s+1:e]) by one warp: the top of the recursion is walked
// by every lane in step, subtrees of at most `span` entries (<= CAP leaves)
// are reduced leaf-parallel.  Result on every lane.
template <int CAP, class T, class G>
__device__ T warp_pw_segment(const G& get, int64_t s, int64_t e, int64_t* loff, int* llen, T* lsum) {
  const int64_t m = e - s - 1;
  if (m <= 0) return get(s);
  constexpr int64_t span = CAP >= 33 ? 4096 : CAP >= 17 ? 2048 : CAP >= 9 ? 1024 : 512;
  const T tail = pw_traverse<T>(
      [&](int64_t lo, int64_t n) { return warp_pw_block<CAP, T>(get, lo, n, loff, llen, lsum); }, s + 1, m, span);
  return get(s) + tail;
}

// LibB / LibC row by one warp (see pw_row_value).  Result on every lane.
template <int CAP, class T, class G>
__device__ T warp_pw_row(const G& get, int64_t s, int64_t e, const int64_t* __restrict__ bounds, int nb,
                         int64_t* loff, int* llen, T* lsum) {
  if (bounds == nullptr) return e == s ? T(0) : warp_pw_segment<CAP, T>(get, s, e, loff, llen, lsum);
  T acc = T(0);
  for (int64_t cur = s, lo = first_bound_after(bounds, nb, s); cur < e; ++lo) {
    const int64_t nxt = (lo < nb && bounds[lo] < e) ? bounds[lo] : e;
    acc = acc + warp_pw_segment<CAP, T>(get, cur, nxt, loff, llen, lsum);
    cur = nxt;
  }
  return acc;
}

// Warp-cooperative L-lane CSR-vector row: lane t < L sums elements t, t+L,
// ... in order, then the halving tree.  The whole warp loads the row in
// coalesced chunks of 4x32 products (all in flight at once); lane t < L then
// takes its elements of each 32-chunk by shuffle (element j of a chunk
// belongs to leaf j % L because L divides 32).  Past-the-end elements are
// +0.0 and leave the (never -0.0) partial sums unchanged.  Result on every
// lane.
template <class T, class G>
__device__ T warp_lane_row(const G& get, int64_t s, int64_t len, int L) {
  const int lane = threadIdx.x & 31;
  T acc = T(0);
  for (int64_t base = 0; base < len; base += 128) {
    T p[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t k = base + c * 32 + lane;
      p[c] = k < len ? get(s + k) : T(0);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (L == 32) {
        acc = acc + p[c];
      } else {
        for (int j = 0; j < 32; j += L) {
          const T q = __shfl_sync(0xffffffffu, p[c], j + (lane & (L - 1)));
          if (lane < L) acc = acc + q;
        }
      }
    }
  }
  for (int h = L >> 1; h >= 1; h >>= 1) {
    const T o = __shfl_down_sync(0xffffffffu, acc, h);
    if (lane < h) acc = acc + o;
  }
  return __shfl_sync(0xffffffffu, acc, 0);
}

// ---------------------------------------------------------------------------
// Row kernel for every row-sorted layout: CSR/LibA/L (kernels.py:167-189),
// CSR/LibB (kernels.py:192-199), CSR/LibC (kernels.py:202-223), COO/LibA
// over the cached run starts (kernels.py:141-153) and the HYB spill
// (kernels.py:262-270, ADD).
//
// The rows are cut once per handle into tiles (RowTile: at most ROWSEG_ROWS
// rows and CAP entries, rows longer than MED_ROW excluded — those are reduced
// first, one CTA each, by cta_long_row).  A persistent CTA (one wave) walks
// its tiles through an NS-deep shared-memory ring:
//   * one thread arms the stage's mbarrier and the TMA engine bulk-copies the
//     tile's row-pointer slice and its vals/cols (16-B aligned supersets,
//     L2 evict-first) into the stage — NS-1 tiles are in flight while one is
//     reduced;
//   * the x gathers of the next tile are issued into registers before the
//     current tile is reduced, and multiplied in place afterwards;
//   * one thread per row reduces it in the configuration's exact order
//     (lane tree / numpy pairwise / chunk pieces); rows longer than the
//     thread limit are reduced by a warp from shared memory.
// ---------------------------------------------------------------------------
struct RowTile {
  long long e0, e1;  // entry range [e0, e1)
  int r0, r1;        // row range [r0, r1)
};
// Stage layout of the ring: vals (products in place), cols, row-pointer slice.
template <class T, class P, int CAP, int NS>
struct PipeLayout {
  static constexpr int PQ = 16 / (int)sizeof(P);  // row-pointer entries per 16 B
  static constexpr size_t SV = (size_t)(CAP + 8) * sizeof(T);
  static constexpr size_t SC = (size_t)(CAP + 8) * 4;
  static constexpr size_t SP = ((size_t)(ROWSEG_ROWS + 1 + 2 * PQ) * sizeof(P) + 15) / 16 * 16;
  static constexpr size_t STAGE = (SV + SC + SP + 127) / 128 * 128;
  static constexpr size_t BYTES = NS * STAGE;
};

template <class T, class P, class L>
__device__ __forceinline__ void issue_tile(unsigned char* stage, uint64_t* bar, const RowTile& t,
                                           const P* __restrict__ ptr, const int* __restrict__ cols,
                                           const T* __restrict__ vals, uint64_t policy) {
  const int64_t pa = t.r0 & ~(int64_t)(L::PQ - 1);
  const int64_t pb = ((int64_t)t.r1 + 1 + L::PQ - 1) & ~(int64_t)(L::PQ - 1);
  const uint32_t np = (uint32_t)((pb - pa) * sizeof(P));
  uint32_t nv = 0, nc = 0;
  int64_t A0 = 0;
  if (t.e1 > t.e0) {
    A0 = t.e0 & ~int64_t(3);
    const int64_t A1 = (t.e1 + 3) & ~int64_t(3);
    nv = (uint32_t)((A1 - A0) * sizeof(T));
    nc = (uint32_t)((A1 - A0) * 4);
  }
  mbar_expect_tx(bar, np + nv + nc);
  bulk_g2s(stage + L::SV + L::SC, ptr + pa, np, bar);
  if (nv) {
    bulk_g2s_hint(stage, vals + A0, nv, bar, policy);
    bulk_g2s_hint(stage + L::SV, cols + A0, nc, bar, policy);
  }
}

// ---------------------------------------------------------------------------
// Rows longer than MED_ROW (a per-handle list): one whole CTA per row, before
// the CTA starts its tiles.  The row's products are staged through the (not
// yet used) ring in chunks of LONG_CHUNK with coalesced loads, all in flight,
// then reduced from shared memory in the configuration's exact order:
//   lane tree  - thread t < L runs leaf t over the chunk (chunk starts are
//                multiples of 32, so leaf membership is k % L), then the
//                halving tree in warp 0;
//   pairwise   - the recursion's top is walked by every thread in step; each
//                subtree of <= LONG_CHUNK addends is staged, its leaves are
//                evaluated by 8-thread groups (one per numpy accumulator),
//                thread 0 combines them along the recursion.
// ---------------------------------------------------------------------------
constexpr int LONG_CHUNK = 2048;
constexpr int LONG_CHUNK_LEAVES = 24;  // leaves of a <= 2048-addend subtree (max 17)

struct LongScratch {
  int64_t loff[LONG_CHUNK_LEAVES];
  int llen[LONG_CHUNK_LEAVES];
  double lsum[LONG_CHUNK_LEAVES];
  double bcast;
  int nleaf;
};

template <class T>
__device__ __forceinline__ void stage_products(T* buf, int64_t lo, int n, const int* __restrict__ cols,
                                               const T* __restrict__ vals, const T* __restrict__ x) {
  constexpr int U = 8;
  for (int i = threadIdx.x; i < n; i += ROWSEG_ROWS * U) {
    T v[U];
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = i + u * ROWSEG_ROWS;
      if (j < n) {
        v[u] = ld_stream(vals + lo + j);
        c[u] = ld_stream(cols + lo + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = i + u * ROWSEG_ROWS;
      if (j < n) buf[j] = v[u] * ld_x(x + c[u]);
    }
  }
}

// pairwise(p[lo : lo+n]), n <= LONG_CHUNK, by the whole CTA; result on all threads
template <class T>
__device__ T cta_pw_block(T* buf, LongScratch* sc, int64_t lo, int64_t n, const int* __restrict__ cols,
                          const T* __restrict__ vals, const T* __restrict__ x) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  stage_products<T>(buf, lo, (int)n, cols, vals, x);
  if (tid == 0) {
    int nl = 0;
    pw_traverse<T>([&](int64_t l, int64_t m) {
      sc->loff[nl] = l - lo;
      sc->llen[nl] = (int)m;
      ++nl;
      return T(0);
    }, lo, n);
    sc->nleaf = nl;
  }
  __syncthreads();
  const int nleaf = sc->nleaf;
  const int grp = lane >> 3, k = lane & 7;
  for (int l0 = warp * 4; l0 < nleaf; l0 += ROWSEG_ROWS / 8) {
    const int li = l0 + grp;
    int b = 0, m = 0;
    if (li < nleaf) {
      b = (int)sc->loff[li];
      m = sc->llen[li];
    }
    T r = T(0);
    if (m >= 8) {
      r = buf[b + k];
      const int lim = m - (m % 8);
      for (int i = 8; i < lim; i += 8) r = r + buf[b + i + k];
    }
    T o = __shfl_down_sync(0xffffffffu, r, 1);
    if ((k & 1) == 0) r = r + o;
    o = __shfl_down_sync(0xffffffffu, r, 2);
    if ((k & 3) == 0) r = r + o;
    o = __shfl_down_sync(0xffffffffu, r, 4);
    if (k == 0) r = r + o;
    if (k == 0 && li < nleaf) {
      if (m < 8) {
        T q = T(-0.0);
        for (int i = 0; i < m; ++i) q = q + buf[b + i];
        r = q;
      } else {
        for (int i = m - (m % 8); i < m; ++i) r = r + buf[b + i];
      }
      sc->lsum[li] = (double)r;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int next = 0;
    sc->bcast = (double)pw_traverse<T>([&](int64_t, int64_t) { return (T)sc->lsum[next++]; }, lo, n);
  }
  __syncthreads();
  const T res = (T)sc->bcast;
  __syncthreads();  // buf and the scratch are reused by the next block
  return res;
}

template <class T, bool ADD, bool LANE>
__device__ void cta_long_row(int row, int64_t s, int64_t e, const int* __restrict__ cols, const T* __restrict__ vals,
                             const T* __restrict__ x, T* __restrict__ y, const int64_t* __restrict__ bounds, int nb,
                             int lanes, T* buf, LongScratch* sc) {
  const int tid = threadIdx.x;
  T v;
  if constexpr (LANE) {
    T acc = T(0);
    for (int64_t base = s; base < e; base += LONG_CHUNK) {
      const int n = (int)(e - base < LONG_CHUNK ? e - base : LONG_CHUNK);
      stage_products<T>(buf, base, n, cols, vals, x);
      __syncthreads();
      if (tid < lanes)
        for (int k = tid; k < n; k += lanes) acc = acc + buf[k];
      __syncthreads();
    }
    if (tid < 32)
      for (int h = lanes >> 1; h >= 1; h >>= 1) {
        const T o = __shfl_down_sync(0xffffffffu, acc, h);
        if (tid < h) acc = acc + o;
      }
    v = acc;
  } else {
    auto get_g = [&](int64_t k) { return ld_stream(vals + k) * ld_x(x + ld_stream(cols + k)); };
    auto segment = [&](int64_t a, int64_t b) {
      const int64_t m = b - a - 1;
      if (m <= 0) return get_g(a);
      const T tail = pw_traverse<T>(
          [&](int64_t lo, int64_t n) { return cta_pw_block<T>(buf, sc, lo, n, cols, vals, x); }, a + 1, m,
          LONG_CHUNK);
      return get_g(a) + tail;
    };
    if (bounds == nullptr) {
      v = segment(s, e);
    } else {
      T acc = T(0);
      for (int64_t cur = s, lo = first_bound_after(bounds, nb, s); cur < e; ++lo) {
        const int64_t nxt = (lo < nb && bounds[lo] < e) ? bounds[lo] : e;
        acc = acc + segment(cur, nxt);
        cur = nxt;
      }
      v = acc;
    }
  }
  if (tid == 0) {
    if (ADD) y[row] = y[row] + v;
    else y[row] = v;
  }
}

// LANE: CSR/LibA/L lane tree; otherwise numpy pairwise (LibB, COO/LibA, HYB
// spill) or chunk pieces (LibC, bounds != nullptr).
// Lane-tree variants with <= 1536-entry tiles fit 5 CTAs per SM when they
// keep <= 96 registers (97 drops them to 4: config 2 CSR/LibA 96 -> 106 us).
template <class T, class P, bool ADD, bool LANE, int CAP, int NS, bool DYN>
__global__ void __launch_bounds__(ROWSEG_ROWS, (LANE && CAP <= 1536) ? 5 : 4) k_rows_pipe(int64_t ntiles, const RowTile* __restrict__ tiles,
                                                           const P* __restrict__ ptr, const int* __restrict__ cols,
                                                           const T* __restrict__ vals, const T* __restrict__ x,
                                                           T* __restrict__ y, const int64_t* __restrict__ bounds,
                                                           int nb, int lanes, int64_t nlong,
                                                           const int* __restrict__ lrow,
                                                           const int64_t* __restrict__ lbeg,
                                                           const int64_t* __restrict__ lend,
                                                           const int* __restrict__ rowmap,
                                                           unsigned long long* __restrict__ ctr) {
  using L = PipeLayout<T, P, CAP, NS>;
  constexpr int U = CAP / ROWSEG_ROWS;  // products per thread per tile (one round of gathers)
  static_assert(CAP % ROWSEG_ROWS == 0 && CAP >= MED_ROW, "tile capacity");
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ alignas(8) uint64_t bar[NS];
  __shared__ RowTile desc[NS];
  __shared__ int64_t sidx[DYN ? NS : 1];   // DYN: tile index each stage holds (>= ntiles: none)
  __shared__ int smed[ROWSEG_ROWS];
  __shared__ int nmed;
  constexpr int NL = LANE ? 1 : MED_LEAVES;
  __shared__ int64_t loff[ROWSEG_ROWS / 32][NL];
  __shared__ int llen[ROWSEG_ROWS / 32][NL];
  __shared__ T lsum[ROWSEG_ROWS / 32][NL];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int thr = LANE ? THREAD_LANE_ROW : THREAD_PW_ROW;
  const uint64_t policy = l2_evict_first_policy();
  if (nlong > 0) {
    static_assert(L::BYTES >= LONG_CHUNK * sizeof(T) + sizeof(LongScratch), "ring too small for long rows");
    T* buf = reinterpret_cast<T*>(ring);
    LongScratch* lsc = reinterpret_cast<LongScratch*>(ring + LONG_CHUNK * sizeof(T));
    for (int64_t li = blockIdx.x; li < nlong; li += gridDim.x) {
      cta_long_row<T, ADD, LANE>(lrow[li], lbeg[li], lend[li], cols, vals, x, y, bounds, nb, lanes, buf, lsc);
      __syncthreads();
    }
  }
  // Tile order: !DYN (regular matrices) round robin, tiles
  // blockIdx.x + k*gridDim.x; DYN (irregular matrices)
  // every CTA claims the next unclaimed tiles once its long rows are done, so
  // a CTA that spent its start on a long row, or whose tiles hold medium
  // rows, takes fewer tiles — with the static order the slowest SM ran 1.6x
  // the average on config 3's HYB spill.  ctr[0] counts claims, ctr[1]
  // finished CTAs; the last CTA resets both, so the next launch on this
  // stream needs no memset.
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    const int64_t first = DYN ? (int64_t)atomicAdd(ctr, (unsigned long long)NS) : 0;
    for (int s = 0; s < NS; ++s) {
      const int64_t ti = DYN ? first + s : blockIdx.x + (int64_t)s * gridDim.x;
      if constexpr (DYN) sidx[s] = ti;
      if (ti < ntiles) {
        desc[s] = tiles[ti];
        issue_tile<T, P, L>(ring + s * L::STAGE, &bar[s], desc[s], ptr, cols, vals, policy);
      }
    }
  }
  __syncthreads();
  // The x gathers of tile i+1 are issued before tile i is reduced, so their
  // latency hides behind the reduction (software pipelining in registers).
  T xv[U];
  int gather_it = 0;
  auto gather = [&](int st) {
    const RowTile& g = desc[st];
    const int gn = (int)(g.e1 - g.e0), goff = (int)(g.e0 - (g.e0 & ~int64_t(3)));
    const int* gsc = reinterpret_cast<const int*>(ring + st * L::STAGE + L::SV);
    mbar_wait(&bar[st], (uint32_t)(gather_it / NS) & 1u);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = tid + u * ROWSEG_ROWS;
      if (j < gn) xv[u] = ld_x(x + gsc[goff + j]);
    }
  };
  // ti: the tile stage it % NS holds (stages are consumed in claim order)
  int64_t ti = DYN ? sidx[0] : (int64_t)blockIdx.x;
  if (ti < ntiles) gather(0);
  for (int it = 0; ti < ntiles; ++it) {
    const int st = it % NS;
    unsigned char* stage = ring + st * L::STAGE;
    T* sv = reinterpret_cast<T*>(stage);
    const P* sp = reinterpret_cast<const P*>(stage + L::SV + L::SC);
    // claim the tile this stage takes next, descriptor fetched early
    int64_t tn = ntiles;
    RowTile nxt{};
    if (tid == 0) {
      tn = DYN ? (int64_t)atomicAdd(ctr, 1ull) : ti + (int64_t)NS * gridDim.x;
      if (tn < ntiles) nxt = tiles[tn];
    }
    const RowTile t = desc[st];
    const int64_t pa = t.r0 & ~(int64_t)(L::PQ - 1);
    const int64_t A0 = t.e0 & ~int64_t(3);
    const int n = (int)(t.e1 - t.e0), off = (int)(t.e0 - A0);
    if (tid == 0) nmed = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = tid + u * ROWSEG_ROWS;
      if (j < n) sv[off + j] = sv[off + j] * xv[u];
    }
    __syncthreads();
    // the next stage's claim was written at least one barrier ago
    const int64_t tnext = DYN ? sidx[(it + 1) % NS] : ti + gridDim.x;
    if (tnext < ntiles) {
      gather_it = it + 1;
      gather((it + 1) % NS);
    }
    auto get_s = [&](int64_t k) { return sv[(int)(k - A0)]; };
    const int nr = t.r1 - t.r0;
    const bool mine = tid < nr;
    const int64_t s = mine ? (int64_t)sp[t.r0 + tid - pa] : 0;
    const int64_t e = mine ? (int64_t)sp[t.r0 + tid + 1 - pa] : 0;
    const int len = (int)(e - s);
    const bool thread_row = mine && len <= thr;
    if (mine && !thread_row) smed[atomicAdd(&nmed, 1)] = tid;
    T v = T(0);
    if constexpr (LANE) {
      const int wmax = __reduce_max_sync(0xffffffffu, thread_row ? len : 0);
      const int base = (int)(s - A0);
      if (thread_row) v = lane_tree_warp<T>([&](int k) { return sv[base + k]; }, len, lanes, wmax);
    } else {
      if (thread_row) v = pw_row_value<T>(get_s, s, e, bounds, nb);
    }
    // tile rows are matrix rows, or (HYB spill) compacted runs mapped to rows
    const int64_t row = rowmap ? (int64_t)(mine ? rowmap[t.r0 + tid] : 0) : (int64_t)t.r0 + tid;
    if (thread_row) {
      if (!ADD) y[row] = v;
      else if (len > 0) y[row] = y[row] + v;   // HYB spill: rows with entries only
    }
    __syncthreads();
    for (int i = warp; i < nmed; i += ROWSEG_ROWS / 32) {
      const int rr = smed[i];
      const int64_t s2 = sp[t.r0 + rr - pa], e2 = sp[t.r0 + rr + 1 - pa];
      T w;
      if constexpr (LANE) w = warp_lane_row<T>(get_s, s2, e2 - s2, lanes);
      else w = warp_pw_row<MED_LEAVES, T>(get_s, s2, e2, bounds, nb, loff[warp], llen[warp], lsum[warp]);
      if (lane == 0) {
        const int64_t yr = rowmap ? (int64_t)rowmap[t.r0 + rr] : (int64_t)t.r0 + rr;
        if (!ADD) y[yr] = w;
        else y[yr] = y[yr] + w;
      }
    }
    __syncthreads();  // stage st and the medium-row list are free again
    if (tid == 0) {
      if constexpr (DYN) sidx[st] = tn;
      if (tn < ntiles) {
        fence_proxy_async_smem();
        desc[st] = nxt;
        issue_tile<T, P, L>(stage, &bar[st], nxt, ptr, cols, vals, policy);
      }
    }
    ti = tnext;
  }
  if (DYN && tid == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

// Tiles of a row pointer: each 128-row block is cut greedily into runs of
// rows of at most `cap` entries, skipping rows longer than MED_ROW.  Pass 1
// (out == nullptr) counts per block, pass 2 writes at the scanned offsets.
template <class P>
__global__ void k_make_tiles(int64_t nrows, const P* __restrict__ ptr, int64_t cap, int64_t* __restrict__ counts,
                             const int64_t* __restrict__ offs, RowTile* __restrict__ out) {
  const int64_t nblk = (nrows + ROWSEG_ROWS - 1) / ROWSEG_ROWS;
  for (int64_t blk = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; blk < nblk;
       blk += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = blk * ROWSEG_ROWS, end = b0 + ROWSEG_ROWS < nrows ? b0 + ROWSEG_ROWS : nrows;
    int64_t cnt = 0, a = b0;
    while (true) {
      while (a < end && (int64_t)ptr[a + 1] - (int64_t)ptr[a] > MED_ROW) ++a;
      if (a >= end) break;
      const int64_t ea = ptr[a];
      int64_t b = a;
      while (b < end && (int64_t)ptr[b + 1] - (int64_t)ptr[b] <= MED_ROW && (int64_t)ptr[b + 1] - ea <= cap) ++b;
      if (out) out[offs[blk] + cnt] = RowTile{ea, (long long)ptr[b], (int)a, (int)b};
      ++cnt;
      a = b;
    }
    if (!out) counts[blk] = cnt;
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

// The same order with S a compile-time constant (S <= 16, the usual worker
// counts): the row's columns are swept in increasing k, CH*S at a time with
// every load issued before the adds (>= 4 columns in flight, as k_ell_sweep),
// column k added to partial k % S — each partial still sees its columns in
// increasing k.  (The loop above keeps one load pair in flight per thread:
// 0.49-0.56 of peak on configs 1-2.)
template <class T, int S>
__global__ void __launch_bounds__(256) k_ell_strided_c(int64_t nrows, int64_t ncols, int64_t width,
                                                       const int* __restrict__ cols, const T* __restrict__ vals,
                                                       const T* __restrict__ x, T* __restrict__ y) {
  constexpr int CH = S >= 4 ? 1 : 4 / S;   // S-column chunks per step
  constexpr int W = CH * S;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    T part[S];
#pragma unroll
    for (int u = 0; u < S; ++u) part[u] = T(0);
    int64_t k = 0;
    for (; k + W <= width; k += W) {
      T v[W], xv[W];
#pragma unroll
      for (int u = 0; u < W; ++u) {
        const int c = ld_stream(cols + (k + u) * nrows + i);
        v[u] = ld_stream(vals + (k + u) * nrows + i);
        xv[u] = c < ncols ? ld_x(x + c) : T(0);
      }
#pragma unroll
      for (int u = 0; u < W; ++u) part[u % S] = part[u % S] + v[u] * xv[u];
    }
#pragma unroll
    for (int u = 0; u < W; ++u) {   // tail: k is a multiple of S here
      if (k + u < width) {
        const int c = ld_stream(cols + (k + u) * nrows + i);
        const T v = ld_stream(vals + (k + u) * nrows + i);
        part[u % S] = part[u % S] + v * (c < ncols ? ld_x(x + c) : T(0));
      }
    }
    T acc = T(0);
#pragma unroll
    for (int u = 0; u < S; ++u) acc = acc + part[u];
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

// ---------------------------------------------------------------------------
// DIA/LibA, offsets in the parameter space (the default for <= 32 stored
// diagonals).  k_dia is latency-bound (ncu, config 5: long-scoreboard
// stalls, DRAM 70 %, L2 48 %): each group of 4 diagonals first loads its
// offsets, then data and x, then waits.  Here the offsets travel in the
// kernel's parameter space (constant bank: nothing on the load chain) and
// the diagonals go in groups of G = 3 — for a stencil the dx = -1, 0, +1
// triple, whose x loads hit the same L1 lines back to back.  Measured at
// config 5 (profiles/r2_dia_variants.json): 8.38 ms vs 8.83 ms for k_dia
// (0.93 vs 0.88 of the copy-bandwidth peak; the 27-stream read ceiling
// measured by profiles/mb_streams.cu is 6.87 TB/s); deeper groups (6, 9),
// two rows per thread, per-CTA row blocks and a TMA-staged ring (tiles of
// every diagonal bulk-copied to shared memory, x gathered by 8 consumer
// warps) were all slower (4.1-5.6 TB/s).  With DOT the dot(dsrc, y) that
// follows the SpMV in CG is folded in (per-CTA partials, fixed-order fold by
// the last CTA; `accumulate` adds into *out).  Per-row operation order as
// k_dia, so y is bit-identical.
// ---------------------------------------------------------------------------
struct DiaOffs {
  long long o[32];
};
constexpr int DIA_REG_MAX = 32;

// RPT rows per thread (i, i + 256, ...) keeps RPT rows' loads in flight.
// (Measured for fp32 at config 2: RPT = 4 did not help — the 4-byte
// requests, not the loads in flight, bound it; see k_dia_f32x4.)
template <class T, int G, bool DOT, int RPT = 1>
__global__ void __launch_bounds__(256) k_dia_reg(int64_t nrows, int64_t ncols, int ndiag, DiaOffs offs,
                                                 const T* __restrict__ data, const T* __restrict__ x,
                                                 T* __restrict__ y, const T* __restrict__ dsrc, double* partials,
                                                 unsigned* counter, double* out, const int* skip, int accumulate) {
  if (DOT && skip != nullptr && *skip) return;
  double dot = 0.0;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x * RPT + threadIdx.x; i0 < nrows;
       i0 += (int64_t)gridDim.x * blockDim.x * RPT) {
    T acc[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc[r] = T(0);
    for (int k0 = 0; k0 < ndiag; k0 += G) {
      T dv[G][RPT], xv[G][RPT];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int k = k0 + u;
        if (k < ndiag) {
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int64_t i = i0 + r * (int64_t)blockDim.x;
            const int64_t j = i + offs.o[k];
            const bool in = i < nrows && j >= 0 && j < ncols;
            dv[u][r] = i < nrows ? ld_stream(data + (int64_t)k * nrows + i) : T(0);
            xv[u][r] = in ? ld_x(x + j) : T(0);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int k = k0 + u;
        if (k < ndiag) {
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int64_t j = i0 + r * (int64_t)blockDim.x + offs.o[k];
            if (j >= 0 && j < ncols) acc[r] = acc[r] + dv[u][r] * xv[u][r];
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int64_t i = i0 + r * (int64_t)blockDim.x;
      if (i < nrows) {
        y[i] = acc[r];
        if (DOT) dot = dot + (double)dsrc[i] * (double)acc[r];
      }
    }
  }
  if (!DOT) return;
  __shared__ double sh[8];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane == 0) sh[wid] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < 8; ++w) b += sh[w];
    partials[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;   // fixed-order fold of the CTA partials by the whole CTA
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(partials + b);
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  if (lane == 0) sh[wid] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int w = 0; w < 8; ++w) g += sh[w];
    *out = accumulate ? *out + g : g;
    *counter = 0;
  }
}

// fp32 DIA with 16-byte requests: one thread per 4 consecutive rows, the
// diagonal's data as one float4 (needs nrows % 4 == 0) and x[i+off ..
// i+off+3] as one float4 when off % 4 == 0, else from the two aligned float4
// around it (the neighbouring threads' lines: L1 hits).  Row groups whose
// window leaves [0, ncols) use scalar loads.  Per row the same ascending-
// diagonal sum as k_dia (skipped cells not added), so y is bit-identical to
// the scalar fp32 kernel.  (4-byte requests held fp32 DIA at 0.48 of peak on
// config 2 — slower in absolute time than fp64.)
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float f4_at(const float4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}
__global__ void __launch_bounds__(256) k_dia_f32x4(int64_t nrows, int64_t ncols, int ndiag, DiaOffs offs,
                                                   const float* __restrict__ data, const float* __restrict__ x,
                                                   float* __restrict__ y) {
  const int64_t ngroups = nrows / 4;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < ngroups;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = gi * 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < ndiag; ++k) {
      const int64_t off = offs.o[k];
      const int64_t j = i + off;
      const float4 dv = ld_stream4(data + (int64_t)k * nrows + i);
      float xv[4];
      const int r = (int)(((j % 4) + 4) % 4);
      const int64_t base = j - r;
      if (base >= 0 && base + 8 <= ncols) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(x + base));
        if (r == 0) {
          xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
        } else {
          const float4 b = __ldg(reinterpret_cast<const float4*>(x + base + 4));
#pragma unroll
          for (int u = 0; u < 4; ++u) xv[u] = r + u < 4 ? f4_at(a, r + u) : f4_at(b, r + u - 4);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = acc[u] + f4_at(dv, u) * xv[u];
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t ju = j + u;
          if (ju >= 0 && ju < ncols) acc[u] = acc[u] + f4_at(dv, u) * __ldg(x + ju);
        }
      }
    }
    *reinterpret_cast<float4*>(y + i) = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
}

// Grid of a grid-stride kernel sized by its real occupancy: grid_for()'s
// 8 CTAs/SM assumes <= 32 registers; a kernel that fits fewer would leave a
// partial second wave doing a full share of the rows (measured: the fused
// DIA SpMV+dot at 36 registers ran 20 % slower on a 1184-CTA grid).
static unsigned resident_grid(const void* kern, int block, int64_t items) {
  static std::mutex mu;
  static std::map<const void*, int> occ;
  int per = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ.find(kern);
    if (it == occ.end()) {
      SVB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, block, 0));
      occ[kern] = per = per < 1 ? 1 : per;
    } else {
      per = it->second;
    }
  }
  return grid_for(items, block, per);
}

// SPMVTUNE_DIA=0 pins the thread-per-row k_dia (A/B experiments)
static bool dia_reg_enabled() {
  static const bool on = [] {
    const char* e = getenv("SPMVTUNE_DIA");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool launch_dia_f32x4(const svb_matrix* m, const float* vals, const float* x, float* y, cudaStream_t s);

template <class T, bool DOT>
static bool launch_dia_reg(const svb_matrix* m, const T* vals, const T* x, T* y, const T* dsrc, double* partials,
                           unsigned* counter, double* out, const int* skip, int accumulate, unsigned max_grid,
                           cudaStream_t s) {
  if (!dia_reg_enabled() || m->ndiag < 1 || m->ndiag > DIA_REG_MAX || m->h_offs.size() != (size_t)m->ndiag)
    return false;
  if constexpr (std::is_same<T, float>::value && !DOT) {
    if (launch_dia_f32x4(m, vals, x, y, s)) return true;
  }
  constexpr int RPT = 1;
  const unsigned g = resident_grid((const void*)k_dia_reg<T, 3, DOT, RPT>, 256, (m->nrows + RPT - 1) / RPT);
  if (DOT && g > max_grid) return false;
  DiaOffs o{};
  for (int k = 0; k < m->ndiag; ++k) o.o[k] = m->h_offs[k];
  k_dia_reg<T, 3, DOT, RPT><<<g, 256, 0, s>>>(m->nrows, m->ncols, (int)m->ndiag, o, vals, x, y, dsrc, partials,
                                              counter, out, skip, accumulate);
  return true;
}

// DIA SpMV fused with the Krylov dot product that always follows it in CG
// (q = A p, then p.q): the same per-row sums as k_dia (identical y), plus
// sum_i dsrc[i] * y[i] folded per CTA and, in the last CTA to finish, over the
// CTA partials in fixed order into *out (deterministic run to run).  The
// separate p.q pass over 16n bytes disappears.  `skip` (batched CG's done
// flag) turns the launch into a no-op after convergence.
__global__ void __launch_bounds__(256) k_dia_dot(int64_t nrows, int64_t ncols, int64_t ndiag,
                                                 const long long* __restrict__ offs, const double* __restrict__ data,
                                                 const double* __restrict__ x, double* __restrict__ y,
                                                 const double* __restrict__ dsrc, double* partials, unsigned* counter,
                                                 double* out, const int* skip, int accumulate) {
  if (skip != nullptr && *skip) return;
  double dot = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    int64_t k = 0;
    for (; k + 4 <= ndiag; k += 4) {
      double v[4], xv[4];
      bool in[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + __ldg(offs + k + u);
        in[u] = j >= 0 && j < ncols;
        v[u] = ld_stream(data + (k + u) * nrows + i);
        xv[u] = in[u] ? ld_x(x + j) : 0.0;
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
    dot = dot + dsrc[i] * acc;
  }
  __shared__ double sh[8];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane == 0) sh[wid] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < 8; ++w) b += sh[w];
    partials[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;   // fixed-order fold of the CTA partials by the whole CTA
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(partials + b);
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  if (lane == 0) sh[wid] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int w = 0; w < 8; ++w) g += sh[w];
    *out = accumulate ? *out + g : g;
    *counter = 0;
  }
}

static bool launch_dia_f32x4(const svb_matrix* m, const float* vals, const float* x, float* y, cudaStream_t s) {
  if (m->nrows % 4 != 0 || m->nrows < 4 || (((uintptr_t)vals | (uintptr_t)x | (uintptr_t)y) & 15) != 0) return false;
  const unsigned g = resident_grid((const void*)k_dia_f32x4, 256, m->nrows / 4);
  DiaOffs o{};
  for (int k = 0; k < m->ndiag; ++k) o.o[k] = m->h_offs[k];
  k_dia_f32x4<<<g, 256, 0, s>>>(m->nrows, m->ncols, (int)m->ndiag, o, vals, x, y);
  return true;
}

void launch_dia_dot(const svb_matrix* m, const double* x, double* y, const double* dsrc, double* partials,
                    unsigned* counter, double* out, const int* skip, unsigned max_grid, cudaStream_t s,
                    int accumulate) {
  SVB_REQUIRE(m->fmt == SVB_DIA, SVB_UNSUPPORTED_CONFIG, "fused SpMV+dot needs a DIA matrix");
  const int64_t n = m->nrows;
  if (launch_dia_reg<double, true>(m, ptr<double>(m->vals), x, y, dsrc, partials, counter, out, skip, accumulate,
                                   max_grid, s)) {
    SVB_CHECK_LAUNCH();
    return;
  }
  unsigned g = grid_for(n, 256, 8);   // the same grid as k_dia: full occupancy
  SVB_REQUIRE(g <= max_grid, SVB_INVALID, "fused SpMV+dot: partials buffer too small");
  k_dia_dot<<<g, 256, 0, s>>>(n, m->ncols, m->ndiag, ptr<long long>(m->offs), ptr<double>(m->vals), x, y, dsrc,
                              partials, counter, out, skip, accumulate);
  SVB_CHECK_LAUNCH();
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

// rows of a row pointer longer than MED_ROW -> (row, begin, end) list
template <class P>
__global__ void k_find_long(int64_t nrows, const P* __restrict__ ptr, unsigned long long* count, int* lrow,
                            int64_t* lbeg, int64_t* lend, const int* __restrict__ rowmap = nullptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = ptr[i], e = ptr[i + 1];
    if (e - b > MED_ROW) {
      const unsigned long long k = atomicAdd(count, 1ull);
      lrow[k] = rowmap ? rowmap[i] : (int)i;
      lbeg[k] = b;
      lend[k] = e;
    }
  }
}

__global__ void k_spill_flags(int64_t n, const long long* __restrict__ ptr, int64_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = ptr[i + 1] > ptr[i] ? 1 : 0;
}
__global__ void k_spill_compact(int64_t n, const long long* __restrict__ ptr, const int64_t* __restrict__ pos,
                                long long* __restrict__ runs, int* __restrict__ map, int64_t nruns) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (ptr[i + 1] > ptr[i]) {
      runs[pos[i]] = ptr[i];
      map[pos[i]] = (int)i;
    }
    if (i == n - 1) runs[nruns] = ptr[n];
  }
}

// HYB spill rows with entries, compacted (built once, cached on the handle)
static int64_t hyb_runs(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->nhruns >= 0) return m->nhruns;
  const int64_t n = m->nrows;
  Buf f = alloc((n + 1) * 8, s), pos = alloc((n + 1) * 8, s);
  const unsigned g = grid_for(n, 256);
  k_spill_flags<<<g, 256, 0, s>>>(n, ptr<long long>(m->ptr), ptr<int64_t>(f));
  SVB_CHECK_LAUNCH();
  const int64_t nr = exclusive_scan_total(ptr<int64_t>(f), ptr<int64_t>(pos), n, s);
  m->hruns = alloc((nr + 1) * 8, s);
  m->hmap = alloc((nr > 0 ? nr : 1) * 4, s);
  k_spill_compact<<<g, 256, 0, s>>>(n, ptr<long long>(m->ptr), ptr<int64_t>(pos), ptr<long long>(m->hruns),
                                    ptr<int>(m->hmap), nr);
  SVB_CHECK_LAUNCH();
  SVB_CUDA_TRY(cudaStreamSynchronize(s));
  detach(m->hruns);
  detach(m->hmap);
  m->nhruns = nr;
  return nr;
}

// The handle's long-segment list (built once, cached): CSR rows, COO runs
// (via a derived row pointer) or the HYB spill runs.
static int64_t long_list(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->nlong >= 0) return m->nlong;
  const int64_t entries = m->fmt == SVB_HYB ? m->spill_nnz : m->nnz;
  const int64_t cap = entries / (MED_ROW + 1) + 1;
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
  } else {  // HYB: the compacted spill runs, rows through the run map
    k_find_long<<<grid_for(m->nhruns > 0 ? m->nhruns : 1, 256), 256, 0, s>>>(
        m->nhruns, ptr<long long>(m->hruns), ptr<unsigned long long>(cnt), ptr<int>(m->lrow),
        ptr<int64_t>(m->lbeg), ptr<int64_t>(m->lend), ptr<int>(m->hmap));
    SVB_CHECK_LAUNCH();
  }
  unsigned long long h = 0;
  SVB_CUDA_TRY(cudaMemcpyAsync(&h, cnt->ptr, 8, cudaMemcpyDeviceToHost, s));
  SVB_CUDA_TRY(cudaStreamSynchronize(s));
  m->nlong = (int64_t)h;
  return m->nlong;
}

// The handle's row tiles (built once per capacity, cached) over its row
// pointer: CSR rows, COO runs (derived pointer) or the HYB spill rows.
template <class P>
static int64_t tile_list(const svb_matrix* m, const P* rp, int cap, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->ntiles >= 0 && m->tile_cap == cap) return m->ntiles;
  const int64_t nrows = m->fmt == SVB_HYB ? m->nhruns : m->nrows;   // HYB: compacted spill runs
  const int64_t nblk = (nrows + ROWSEG_ROWS - 1) / ROWSEG_ROWS;
  Buf cnt = alloc((nblk + 1) * 8, s), off = alloc((nblk + 1) * 8, s);
  const unsigned g = grid_for(nblk, 128);
  k_make_tiles<P><<<g, 128, 0, s>>>(nrows, rp, cap, ptr<int64_t>(cnt), nullptr, nullptr);
  SVB_CHECK_LAUNCH();
  const int64_t total = exclusive_scan_total(ptr<int64_t>(cnt), ptr<int64_t>(off), nblk, s);
  Buf tiles = alloc((total > 0 ? total : 1) * sizeof(RowTile), s);
  if (total > 0) {
    k_make_tiles<P><<<g, 128, 0, s>>>(nrows, rp, cap, nullptr, ptr<int64_t>(off), ptr<RowTile>(tiles));
    SVB_CHECK_LAUNCH();
  }
  SVB_CUDA_TRY(cudaStreamSynchronize(s));  // an older tile list may still be in use elsewhere
  detach(tiles);
  m->tiles = tiles;
  m->tile_cap = cap;
  m->ntiles = total;
  return total;
}

// Per-(handle, stream) counters of the row kernel's dynamic tile scheduler
// (zeroed once here, reset by the last CTA of every launch; launches on one
// stream are serialised, so they never share a live counter).
static unsigned long long* tile_counter(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  for (auto& e : m->tctr)
    if (e.first == s) return ptr<unsigned long long>(e.second);
  Buf b = alloc(16, s);
  SVB_CUDA_TRY(cudaMemsetAsync(b->ptr, 0, 16, s));
  detach(b);
  m->tctr.emplace_back(s, b);
  return ptr<unsigned long long>(b);
}

template <class T, class P, bool ADD, bool LANE, int CAP, int NS, bool DYN>
static void launch_rows_kernel(const svb_matrix* m, int64_t nt, int64_t nl, const P* rp, const int* cols,
                               const T* vals, const T* x, T* y, const int64_t* bounds, int nb, int lanes,
                               cudaStream_t s) {
  using L = PipeLayout<T, P, CAP, NS>;
  auto* kern = k_rows_pipe<T, P, ADD, LANE, CAP, NS, DYN>;
  static const int occ = [kern] {
    SVB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES));
    int o = 0;
    SVB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, ROWSEG_ROWS, L::BYTES));
    return o < 1 ? 1 : o;
  }();
  const int64_t work = nt > nl ? nt : nl;
  const int64_t cap = (int64_t)sm_count() * occ;
  const unsigned g = (unsigned)(work < cap ? work : cap);
  kern<<<g, ROWSEG_ROWS, L::BYTES, s>>>(nt, ptr<RowTile>(m->tiles), rp, cols, vals, x, y, bounds, nb, lanes, nl,
                                        ptr<int>(m->lrow), ptr<int64_t>(m->lbeg), ptr<int64_t>(m->lend),
                                        m->fmt == SVB_HYB ? ptr<int>(m->hmap) : nullptr,
                                        DYN ? tile_counter(m, s) : nullptr);
  SVB_CHECK_LAUNCH();
}

template <class T, class P, bool ADD, bool LANE, int CAP, int NS>
static void launch_rows_cfg(const svb_matrix* m, const P* rp, const int* cols, const T* vals, const T* x, T* y,
                            const int64_t* bounds, int nb, int lanes, cudaStream_t s) {
  const int64_t nt = tile_list(m, rp, CAP, s);
  const int64_t nl = long_list(m, s);
  if ((nt > nl ? nt : nl) <= 0) return;
  // dynamic tile claims where per-tile work varies: rows longer than
  // MED_ROW exist; the round-robin order stays for regular matrices, where
  // the shared counter cost 2-9 us per launch on configs 1/2
  // (SPMVTUNE_ROWDYN=0/1 forces either order for experiments)
  static const int dyn_env = [] {
    const char* e = getenv("SPMVTUNE_ROWDYN");
    return e ? atoi(e) : -1;
  }();
  if (dyn_env >= 0 ? dyn_env > 0 : nl > 0)
    launch_rows_kernel<T, P, ADD, LANE, CAP, NS, true>(m, nt, nl, rp, cols, vals, x, y, bounds, nb, lanes, s);
  else
    launch_rows_kernel<T, P, ADD, LANE, CAP, NS, false>(m, nt, nl, rp, cols, vals, x, y, bounds, nb, lanes, s);
}

// The persistent row kernel.  The tile capacity follows the mean entries per
// 128-row block (a full stage wastes least ring space); SPMVTUNE_ROWCFG=1..3
// pins a variant for experiments.
template <class T, class P, bool ADD>
static void launch_rows(const svb_matrix* m, const P* rp, const int* cols, const T* vals, const T* x, T* y,
                        const int64_t* bounds, int nb, int lanes, cudaStream_t s) {
  static const int forced = [] {
    const char* e = getenv("SPMVTUNE_ROWCFG");
    return e ? atoi(e) : 0;
  }();
  const int64_t entries = m->fmt == SVB_HYB ? m->spill_nnz : m->nnz;
  const int64_t trows = m->fmt == SVB_HYB ? m->nhruns : m->nrows;   // HYB: compacted spill runs
  const double per_block = trows > 0 ? (double)entries * ROWSEG_ROWS / (double)trows : 0.0;
  // Irregular row lengths (some row longer than MED_ROW, e.g. power-law):
  // the gathers and the per-row reductions, not the stream, bound the
  // kernel, and smaller tiles (more CTAs per SM) win — measured on a 4 M-row
  // power-law matrix: CSR 1536-entry tiles 12-22 % faster than 2048, COO
  // runs 1024-entry tiles 14 % faster.
  const bool irregular = long_list(m, s) > 0;
  int cfg = per_block <= 900 ? 3 : per_block <= 1400 ? 1 : 2;
  if (irregular && m->fmt == SVB_CSR && cfg == 2) cfg = 1;
  if (irregular && m->fmt == SVB_COO) cfg = 3;
  if (forced) cfg = forced;
  auto go = [&](auto lane_tag) {
    constexpr bool LANE = decltype(lane_tag)::value;
    switch (cfg) {
      case 3: launch_rows_cfg<T, P, ADD, LANE, 1024, 3>(m, rp, cols, vals, x, y, bounds, nb, lanes, s); break;
      case 1: launch_rows_cfg<T, P, ADD, LANE, 1536, 2>(m, rp, cols, vals, x, y, bounds, nb, lanes, s); break;
      default: launch_rows_cfg<T, P, ADD, LANE, 2048, 2>(m, rp, cols, vals, x, y, bounds, nb, lanes, s); break;
    }
  };
  if (lanes > 0) go(std::true_type{});
  else go(std::false_type{});
}

template <class T>
static void launch_spmv(const svb_matrix* m, int fmt, int lib, int lane, int workers,
                        const T* vals, const T* svals, const T* x, T* y, cudaStream_t s) {
  const int64_t n = m->nrows;
  // the row kernel's bulk copies need 16-B aligned bases (every buffer of a
  // handle comes from svb::alloc, which guarantees it)
  for (const void* p : {(const void*)vals, (const void*)svals, (const void*)ptr<int>(m->cols),
                        (const void*)ptr<int>(m->scols)})
    SVB_REQUIRE(((uintptr_t)p & 15) == 0, SVB_INVALID, "matrix buffers must be 16-byte aligned");
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
    if (m->ptr64)
      launch_rows<T, long long, false>(m, ptr<long long>(m->ptr), ptr<int>(m->cols), vals, x, y, bounds, nb, lanes, s);
    else
      launch_rows<T, int, false>(m, ptr<int>(m->ptr), ptr<int>(m->cols), vals, x, y, bounds, nb, lanes, s);
    return;
  } else if (fmt == SVB_COO) {
    if (lib == SVB_LIBA) {
      // row runs of the sorted coordinates (kernels.py:141-153), reduced in
      // reduceat order by the row kernel; rows without entries get 0
      const long long* runs = coo_runs(m, s);
      launch_rows<T, long long, false>(m, runs, ptr<int>(m->cols), vals, x, y, nullptr, 0, 0, s);
      return;
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
      const unsigned g = grid_for(n, 256, 8);
      const int* ec = ptr<int>(m->cols);
      // S >= width: one column per partial, i.e. the plain column sweep's
      // sums (0 + p is p; the partials start from +0.0)
      if (S >= m->width) {
        k_ell_sweep<T><<<g, 256, 0, s>>>(n, m->ncols, m->width, ec, vals, x, y);
      } else {
        switch (S) {
#define SVB_ELLC(K) \
  case K:           \
    k_ell_strided_c<T, K><<<g, 256, 0, s>>>(n, m->ncols, m->width, ec, vals, x, y); \
    break;
          SVB_ELLC(1) SVB_ELLC(2) SVB_ELLC(3) SVB_ELLC(4) SVB_ELLC(5) SVB_ELLC(6) SVB_ELLC(7) SVB_ELLC(8)
          SVB_ELLC(9) SVB_ELLC(10) SVB_ELLC(11) SVB_ELLC(12) SVB_ELLC(13) SVB_ELLC(14) SVB_ELLC(15) SVB_ELLC(16)
#undef SVB_ELLC
          default: k_ell_strided<T><<<g, 256, 0, s>>>(n, m->ncols, m->width, S, ec, vals, x, y);
        }
      }

    }
  } else if (fmt == SVB_DIA) {
    if (!launch_dia_reg<T, false>(m, vals, x, y, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, s))
      k_dia<T><<<grid_for(n, 256, 8), 256, 0, s>>>(n, m->ncols, m->ndiag, ptr<long long>(m->offs), vals, x, y);
  } else {  // HYB
    k_ell_sweep<T><<<grid_for(n, 256, 8), 256, 0, s>>>(n, m->ncols, m->width, ptr<int>(m->cols), vals, x, y);
    SVB_CHECK_LAUNCH();
    if (m->spill_nnz > 0) {
      hyb_runs(m, s);
      launch_rows<T, long long, true>(m, ptr<long long>(m->hruns), ptr<int>(m->scols), svals, x, y, nullptr, 0, 0,
                                      s);
    }
    return;
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
