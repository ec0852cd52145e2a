// Device-resident sparse matrix handle (the svb_matrix behind the C ABI).
//
// One struct covers the five reference containers (formats.py:50-260).  All
// buffers are immutable once the handle is published, so conversions share
// them freely (CSR->COO reuses col/val buffers; COO->CSR likewise).
#pragma once

#include <mutex>
#include <vector>

#include "common.cuh"

struct svb_matrix {
  int fmt = SVB_CSR;
  int64_t nrows = 0, ncols = 0, nnz = 0;
  bool ptr64 = false;      // row pointer element type on device
  int64_t width = 0;       // ELL / HYB-ELL width
  int64_t ndiag = 0;       // DIA
  int64_t spill_nnz = 0;   // HYB COO part

  svb::Buf ptr;    // CSR row_ptr (int32/int64) [nrows+1]; HYB: spill row_ptr (int64)
  svb::Buf rows;   // COO rows int32 [nnz]; HYB spill rows int32
  svb::Buf cols;   // CSR/COO cols int32 [nnz]; ELL/HYB cols int32 [width*nrows]
  svb::Buf vals;   // f64 values in the layout of `cols`; DIA data [ndiag*nrows]
  svb::Buf offs;   // DIA offsets int64 [ndiag]
  svb::Buf scols;  // HYB spill cols int32
  svb::Buf svals;  // HYB spill values f64
  std::vector<int64_t> h_offs;  // DIA offsets on the host (kernel launch args)

  // lazily created fp32 copies of the value arrays (SVB_F32 SpMV)
  mutable std::mutex mu;
  mutable svb::Buf vals32, svals32;
  // rows/runs longer than LONG_ROW (CSR rows, COO runs, HYB spill runs):
  // (row, first entry, end) lists built on first use by the SpMV dispatcher
  mutable int64_t nlong = -1;
  mutable svb::Buf lrow, lbeg, lend;
  // row tiles of the staged row kernel (spmv.cu RowTile), built on first use
  mutable int64_t ntiles = -1;
  mutable int tile_cap = 0;  // entry capacity the tiles were cut for
  mutable svb::Buf tiles;
  // the row kernel's dynamic tile counters, one per launching stream
  mutable std::vector<std::pair<cudaStream_t, svb::Buf>> tctr;
  // COO: row-run starts (int64 row pointer derived from the sorted rows —
  // what np.flatnonzero(np.diff(rows)) computes on every reference call)
  mutable svb::Buf dptr;
  // HYB: the spill rows that have entries, compacted (run pointer int64
  // [nhruns+1] into the spill arrays, row of each run int32 [nhruns]), so
  // the spill kernel never tiles the rows that spill nothing
  mutable int64_t nhruns = -1;
  mutable svb::Buf hruns, hmap;
  // CSR: the diagonal-occupancy bitmap svb_features built (bit c - i + n - 1),
  // reused by the DIA conversion instead of a second pass over col_idx
  mutable svb::Buf diag_bits;
  // ... and the sorted diagonal offsets of that bitmap when there are at
  // most DIA_OFFSET_CAP of them (the DIA conversion skips its offset scan)
  mutable bool diag_offs_valid = false;
  mutable std::vector<int64_t> diag_offs;

  int64_t device_bytes() const {
    int64_t b = 0;
    const svb::Buf* all[] = {&ptr, &rows, &cols, &vals, &offs, &scols, &svals, &vals32, &svals32};
    for (const svb::Buf* p : all)
      if (*p) b += (int64_t)(*p)->bytes;
    return b;
  }
};

namespace svb {

// Long-lived buffers are freed on the legacy stream after a device-wide sync
// (svb_matrix_destroy), never on the stream that allocated them: that stream
// may belong to a thread (the advisor) that is gone by then.
inline void detach(Buf& b) {
  if (b) b->stream = 0;
}
inline svb_matrix* publish(svb_matrix* m) {
  for (Buf* b : {&m->ptr, &m->rows, &m->cols, &m->vals, &m->offs, &m->scols, &m->svals}) detach(*b);
  return m;
}

// fp32 copies of vals / svals, created on first use on `s`
const float* vals_f32(const svb_matrix* m, cudaStream_t s);
const float* svals_f32(const svb_matrix* m, cudaStream_t s);

// helpers shared by the conversion and feature code
void narrow_i64_to_i32(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s);
void widen_i32_to_i64(const int32_t* src, int64_t* dst, int64_t n, cudaStream_t s);
void ptr_to_i64(const svb_matrix* m, int64_t* dst, cudaStream_t s);  // CSR row_ptr -> int64
Buf upload(const void* host, size_t bytes, cudaStream_t s);
Buf rows_to_ptr(const int32_t* rows, int64_t nnz, int64_t nrows, bool ptr64, cudaStream_t s);
Buf ptr_to_rows(const svb_matrix* m, cudaStream_t s);
void forget_bounds(const svb_matrix* m);  // drop cached LibC chunk bounds (spmv.cu)
// DIA SpMV y = A x fused with sum dsrc.y into *out (spmv.cu, k_dia_dot);
// partials holds >= max_grid doubles, counter is zero and left zero
void launch_dia_dot(const svb_matrix* m, const double* x, double* y, const double* dsrc, double* partials,
                    unsigned* counter, double* out, const int* skip, unsigned max_grid, cudaStream_t s,
                    int accumulate = 0);
// y = A x in any configuration (the svb_spmv dispatcher)
void spmv_dispatch(const svb_matrix* m, int fmt, int lib, int lane, int workers, int dtype, const void* x, void* y,
                   cudaStream_t s);

// exclusive scan of int64 counts (n+1 outputs; out[n] = total) and the total
// copied back to the host (synchronises `s`)
int64_t exclusive_scan_total(const int64_t* counts, int64_t* out, int64_t n, cudaStream_t s);

// ---------------------------------------------------------------------------
// Row tiles staged through shared memory.  Thread-per-row kernels over CSR
// read col_idx with a stride of one row per lane (poorly coalesced); a CTA
// instead copies the contiguous nnz range of its BLOCK rows into shared
// memory with coalesced loads and lets each thread walk its row there.
// Tiles whose nnz exceed the capacity are walked straight from global
// memory (staged == false).  Call from every thread of the CTA.
// ---------------------------------------------------------------------------
template <class P>
struct StagedRows {
  int64_t r0, r1, base;
  bool staged;
};

template <class P, int BLOCK, int CAP>
__device__ __forceinline__ StagedRows<P> stage_row_tile(int64_t tile, int64_t nrows, const P* __restrict__ ptr,
                                                     const int* __restrict__ cols, int* scols,
                                                     const double* __restrict__ vals = nullptr,
                                                     double* svals = nullptr) {
  StagedRows<P> t;
  t.r0 = tile * BLOCK;
  t.r1 = t.r0 + BLOCK < nrows ? t.r0 + BLOCK : nrows;
  t.base = (int64_t)ptr[t.r0];
  const int64_t cnt = (int64_t)ptr[t.r1] - t.base;
  t.staged = cnt <= CAP;
  __syncthreads();  // the previous tile's readers are done with the buffers
  if (t.staged) {
    for (int64_t k = threadIdx.x; k < cnt; k += BLOCK) {
      scols[k] = __ldg(cols + t.base + k);
      if (svals) svals[k] = __ldg(vals + t.base + k);
    }
  }
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------
// Row-tile ring: fixed R-row tiles (tile t = rows [tR, min((t+1)R, n))) whose
// row-pointer slice and, when the tile's entries fit CAP, col_idx range
// (and optionally the values) are bulk-copied (TMA engine, mbarrier
// completion) into an NS-stage shared-memory ring by one thread, so NS-1
// tiles are in flight while one is walked.  The synchronous stage_row_tile
// keeps one 4-byte load per thread in flight; the ring keeps ~NS x 10-40 KB
// per CTA in flight, which is what HBM needs (Little's law: ~45 KB per SM).
// Copies are 16-B aligned supersets (device buffers carry a 128-B tail).
// ---------------------------------------------------------------------------
template <class P, int R, int CAP, bool VALS>
struct RingLayout {
  static constexpr size_t SV = VALS ? (size_t)(CAP + 8) * 8 : 0;
  static constexpr size_t SC = (size_t)(CAP + 8) * 4;
  static constexpr size_t SP = ((size_t)(R + 1) * sizeof(P) + 32 + 15) / 16 * 16;
  static constexpr size_t STAGE = (SV + SC + SP + 127) / 128 * 128;
};

struct RingDesc {
  int64_t r0, r1, e0, e1;  // rows [r0, r1), entries [e0, e1)
  int poff, coff, voff;    // element offsets of r0 / e0 inside the staged supersets
  int staged;              // entries [e0, e0 + staged) are in shared memory, the rest in global
};

__device__ __forceinline__ uintptr_t align_dn16(const void* p) { return (uintptr_t)p & ~(uintptr_t)15; }
__device__ __forceinline__ uintptr_t align_up16(const void* p) {
  return ((uintptr_t)p + 15) & ~(uintptr_t)15;
}

// One thread: arm `bar` and bulk-copy tile [r0, r1) (entries [e0, e1)) into
// `stage`.  The entries are staged up to the stage's capacity: a tile whose
// entries overflow it keeps its first d->staged entries in shared memory and
// the readers take the rest from global memory (a power-law tile with one
// long row no longer drops the whole tile to uncoalesced reads).
template <class P, int R, int CAP, bool VALS>
__device__ __forceinline__ void ring_issue(unsigned char* stage, uint64_t* bar, RingDesc* d, int64_t r0, int64_t r1,
                                           int64_t e0, int64_t e1, const P* ptr, const int* cols,
                                           const double* vals, uint64_t policy) {
  using Lay = RingLayout<P, R, CAP, VALS>;
  const uintptr_t pa = align_dn16(ptr + r0);
  const uint32_t np = (uint32_t)(align_up16(ptr + r1 + 1) - pa);
  uint32_t nc = 0, nv = 0;
  uintptr_t ca = 0, va = 0;
  int coff = 0, voff = 0;
  int64_t nst = 0;
  if (e1 > e0) {
    ca = align_dn16(cols + e0);
    coff = (int)(((uintptr_t)(cols + e0) - ca) / 4);
    nst = e1 - e0;
    nst = nst < (int64_t)(Lay::SC / 4) - coff ? nst : (int64_t)(Lay::SC / 4) - coff;
    if (VALS) {
      va = align_dn16(vals + e0);
      voff = (int)(((uintptr_t)(vals + e0) - va) / 8);
      nst = nst < (int64_t)(Lay::SV / 8) - voff ? nst : (int64_t)(Lay::SV / 8) - voff;
    }
    nc = (uint32_t)(align_up16(cols + e0 + nst) - ca);
    if (VALS) nv = (uint32_t)(align_up16(vals + e0 + nst) - va);
  }
  *d = RingDesc{r0, r1, e0, e1, (int)(((uintptr_t)(ptr + r0) - pa) / sizeof(P)), coff, voff, (int)nst};
  mbar_expect_tx(bar, np + nc + nv);
  bulk_g2s(stage + Lay::SV + Lay::SC, reinterpret_cast<const void*>(pa), np, bar);
  if (nc) bulk_g2s_hint(stage + Lay::SV, reinterpret_cast<const void*>(ca), nc, bar, policy);
  if (nv) bulk_g2s_hint(stage, reinterpret_cast<const void*>(va), nv, bar, policy);
}

// Diagonal-occupancy bitmap marking with a per-CTA cache of
// diagonal indices already set: a stencil or banded matrix touches a handful
// of diagonals, so nearly every entry hits the cache and the global bitmap
// sees one atomicOr per (CTA, diagonal) instead of one per entry.  D is the
// diagonal-index type: 32-bit whenever nrows + ncols - 1 < 2^32 (every
// matrix with int32 columns and at most 2^31 rows), 64-bit otherwise; the
// empty slot is D(-1), never a valid index.
constexpr int DIAG_CACHE = 512;
template <class D>
__device__ __forceinline__ void diag_cache_init(D* cache) {
  for (int k = threadIdx.x; k < DIAG_CACHE; k += blockDim.x) cache[k] = D(-1);
}
// The cache is 4-way set-associative: 128 sets of 4 diagonals, the set
// index a weighted fold of the diagonal's 9-bit groups.  Stencil diagonals
// sit at multiples of the grid pitch (0, ±1, ±nx, ±nx±1, ±nx², ...); a
// direct-mapped cache indexed by the low bits put three or nine hot
// diagonals on one slot whenever nx or nx² is a multiple of 512 (nx = 512,
// 1024, 2048; 3-D nx = 128), each entry evicted its neighbour's and became a
// same-address global atomic (feature pass of conv-diff 2048²: 9.1 ms
// instead of 0.16; 2-D 5/9-point nx = 200..4200 and 3-D 7/27-point nx =
// 40..720: 245 stencils collided).  With this index no set holds more than
// four of those stencils' diagonals (checked offline over the same ranges);
// any direct-mapped index collides on some of them (27 diagonals in 512
// slots), a multiplicative hash on half of the 27-point ones.
template <class D>
__device__ __forceinline__ int diag_set(D d) {
  static_assert(DIAG_CACHE == 512, "the fold below assumes 128 sets of 4");
  const unsigned long long u = (unsigned long long)d;
  return (int)((u + (u >> 9) * 7 + (u >> 18) * 13 + (u >> 27) * 31) & 127);
}
template <class D>
__device__ __forceinline__ void mark_diag(unsigned* __restrict__ bits, D d, D* cache) {
  D* set = cache + 4 * diag_set(d);
  const volatile D* vs = set;
  const D c0 = vs[0], c1 = vs[1], c2 = vs[2], c3 = vs[3];
  if (c0 == d || c1 == d || c2 == d || c3 == d) return;
  const unsigned m = 1u << (d & 31);
  unsigned* w = bits + (d >> 5);
  // a free way: first use (a stencil's few hot diagonals, every CTA at
  // once) — test before setting, so the diagonal's word sees reads, not
  // thousands of same-address atomics
  const int way = c0 == D(-1) ? 0 : c1 == D(-1) ? 1 : c2 == D(-1) ? 2 : c3 == D(-1) ? 3 : -1;
  if (way >= 0) {
    if (!(*(volatile unsigned*)w & m)) atomicOr(w, m);
    set[way] = d;   // racy but benign: a lost insert only costs a global update
    return;
  }
  // an eviction: diagonals spread over millions of words (power-law) —
  // fire-and-forget (RED, result unused), no L2 round trip on the thread's
  // critical path
  atomicOr(w, m);
  set[(int)(d & 3)] = d;
}

}  // namespace svb
