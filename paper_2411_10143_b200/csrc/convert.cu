// Format conversion on the device: convert(m, target) (formats.py:302-320).
//
// The reference routes every conversion through COO (to_coo, formats.py:
// 281-299).  Here every source is first reduced to a "row view" — an int64
// row pointer plus int32 columns and f64 values in row-major order — which
// CSR and COO sources provide without copying; ELL/DIA/HYB sources are
// expanded by a count -> scan -> fill pass.  Targets are then built from the
// row view.  All index/value arrays are bit-identical to the reference's.
#include <algorithm>
#include <vector>

#include "matrix.cuh"

namespace svb {

struct RowView {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  Buf ptr;   // int64 [nrows+1]
  Buf rows;  // int32 [nnz] (only when already available)
  Buf cols;  // int32 [nnz]
  Buf vals;  // f64 [nnz]
};

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// to row view from ELL / DIA / HYB
// ---------------------------------------------------------------------------
__global__ void k_ell_count(int64_t nrows, int64_t ncols, int64_t width, const int* __restrict__ cols,
                            int64_t* __restrict__ cnt) {
  GRID_STRIDE(i, nrows) {
    int64_t c = 0;
    for (int64_t k = 0; k < width; ++k) c += cols[k * nrows + i] != ncols;
    cnt[i] = c;
  }
}

__global__ void k_ell_fill(int64_t nrows, int64_t ncols, int64_t width, const int* __restrict__ ecols,
                           const double* __restrict__ evals, const int64_t* __restrict__ ptr,
                           int* __restrict__ cols, double* __restrict__ vals) {
  GRID_STRIDE(i, nrows) {
    int64_t o = ptr[i];
    for (int64_t k = 0; k < width; ++k) {
      const int c = ecols[k * nrows + i];
      if (c != ncols) {
        cols[o] = c;
        vals[o] = evals[k * nrows + i];
        ++o;
      }
    }
  }
}

__global__ void k_dia_count(int64_t nrows, int64_t ncols, int64_t ndiag, const long long* __restrict__ offs,
                            const double* __restrict__ data, int64_t* __restrict__ cnt) {
  GRID_STRIDE(i, nrows) {
    int64_t c = 0;
    for (int64_t k = 0; k < ndiag; ++k) {
      const int64_t j = i + offs[k];
      c += (j >= 0 && j < ncols && data[k * nrows + i] != 0.0);
    }
    cnt[i] = c;
  }
}

__global__ void k_dia_fill(int64_t nrows, int64_t ncols, int64_t ndiag, const long long* __restrict__ offs,
                           const double* __restrict__ data, const int64_t* __restrict__ ptr,
                           int* __restrict__ cols, double* __restrict__ vals) {
  GRID_STRIDE(i, nrows) {
    int64_t o = ptr[i];
    for (int64_t k = 0; k < ndiag; ++k) {
      const int64_t j = i + offs[k];
      const double v = data[k * nrows + i];
      if (j >= 0 && j < ncols && v != 0.0) {
        cols[o] = (int)j;
        vals[o] = v;
        ++o;
      }
    }
  }
}

// HYB -> row view: merge the row's ELL cells (k order) with its spill run,
// by column, as from_triplets' lexsort would (formats.py:292-298).
__global__ void k_hyb_count(int64_t nrows, int64_t ncols, int64_t width, const int* __restrict__ ecols,
                            const int64_t* __restrict__ sptr, int64_t* __restrict__ cnt) {
  GRID_STRIDE(i, nrows) {
    int64_t c = sptr[i + 1] - sptr[i];
    for (int64_t k = 0; k < width; ++k) c += ecols[k * nrows + i] != ncols;
    cnt[i] = c;
  }
}

__global__ void k_hyb_fill(int64_t nrows, int64_t ncols, int64_t width, const int* __restrict__ ecols,
                           const double* __restrict__ evals, const int64_t* __restrict__ sptr,
                           const int* __restrict__ scols, const double* __restrict__ svals,
                           const int64_t* __restrict__ ptr, int* __restrict__ cols,
                           double* __restrict__ vals) {
  GRID_STRIDE(i, nrows) {
    int64_t o = ptr[i];
    int64_t k = 0, q = sptr[i];
    const int64_t qe = sptr[i + 1];
    // advance k to the next stored ELL cell
    auto next_k = [&](int64_t kk) {
      while (kk < width && ecols[kk * nrows + i] == ncols) ++kk;
      return kk;
    };
    k = next_k(0);
    while (k < width || q < qe) {
      const bool take_ell = q >= qe || (k < width && ecols[k * nrows + i] < scols[q]);
      if (take_ell) {
        cols[o] = ecols[k * nrows + i];
        vals[o] = evals[k * nrows + i];
        k = next_k(k + 1);
      } else {
        cols[o] = scols[q];
        vals[o] = svals[q];
        ++q;
      }
      ++o;
    }
  }
}

static RowView row_view(const svb_matrix* m, cudaStream_t s) {
  RowView v;
  v.nrows = m->nrows;
  v.ncols = m->ncols;
  const int64_t n = m->nrows;
  if (m->fmt == SVB_CSR) {
    v.nnz = m->nnz;
    v.ptr = alloc((n + 1) * 8, s);
    ptr_to_i64(m, ptr<int64_t>(v.ptr), s);
    v.cols = m->cols;
    v.vals = m->vals;
    return v;
  }
  if (m->fmt == SVB_COO) {
    v.nnz = m->nnz;
    v.ptr = rows_to_ptr(ptr<int32_t>(m->rows), m->nnz, n, true, s);
    v.rows = m->rows;
    v.cols = m->cols;
    v.vals = m->vals;
    return v;
  }
  Buf cnt = alloc(n * 8, s);
  const unsigned g = grid_for(n, 256);
  if (m->fmt == SVB_ELL)
    k_ell_count<<<g, 256, 0, s>>>(n, m->ncols, m->width, ptr<int>(m->cols), ptr<int64_t>(cnt));
  else if (m->fmt == SVB_DIA)
    k_dia_count<<<g, 256, 0, s>>>(n, m->ncols, m->ndiag, ptr<long long>(m->offs), ptr<double>(m->vals),
                                  ptr<int64_t>(cnt));
  else
    k_hyb_count<<<g, 256, 0, s>>>(n, m->ncols, m->width, ptr<int>(m->cols), ptr<int64_t>(m->ptr),
                                  ptr<int64_t>(cnt));
  SVB_CHECK_LAUNCH();
  v.ptr = alloc((n + 1) * 8, s);
  v.nnz = exclusive_scan_total(ptr<int64_t>(cnt), ptr<int64_t>(v.ptr), n, s);
  v.cols = alloc(v.nnz * 4, s);
  v.vals = alloc(v.nnz * 8, s);
  if (m->fmt == SVB_ELL)
    k_ell_fill<<<g, 256, 0, s>>>(n, m->ncols, m->width, ptr<int>(m->cols), ptr<double>(m->vals),
                                 ptr<int64_t>(v.ptr), ptr<int>(v.cols), ptr<double>(v.vals));
  else if (m->fmt == SVB_DIA)
    k_dia_fill<<<g, 256, 0, s>>>(n, m->ncols, m->ndiag, ptr<long long>(m->offs), ptr<double>(m->vals),
                                 ptr<int64_t>(v.ptr), ptr<int>(v.cols), ptr<double>(v.vals));
  else
    k_hyb_fill<<<g, 256, 0, s>>>(n, m->ncols, m->width, ptr<int>(m->cols), ptr<double>(m->vals),
                                 ptr<int64_t>(m->ptr), ptr<int>(m->scols), ptr<double>(m->svals),
                                 ptr<int64_t>(v.ptr), ptr<int>(v.cols), ptr<double>(v.vals));
  SVB_CHECK_LAUNCH();
  return v;
}

// ---------------------------------------------------------------------------
// row statistics used by the builders
// ---------------------------------------------------------------------------
__global__ void k_max_len(int64_t nrows, const int64_t* __restrict__ ptr, unsigned long long* out) {
  int64_t best = 0;
  GRID_STRIDE(i, nrows) best = max(best, ptr[i + 1] - ptr[i]);
  for (int o = 16; o; o >>= 1) best = max(best, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)best);
}

static int64_t max_row_len(const RowView& v, cudaStream_t s) {
  Buf d = alloc(8, s);
  SVB_CUDA_TRY(cudaMemsetAsync(d->ptr, 0, 8, s));
  k_max_len<<<grid_for(v.nrows, 256), 256, 0, s>>>(v.nrows, ptr<int64_t>(v.ptr),
                                                   ptr<unsigned long long>(d));
  SVB_CHECK_LAUNCH();
  unsigned long long h = 0;
  SVB_CUDA_TRY(cudaMemcpyAsync(&h, d->ptr, 8, cudaMemcpyDeviceToHost, s));
  SVB_CUDA_TRY(cudaStreamSynchronize(s));
  return (int64_t)h;
}

// row-length histogram, privatised in shared memory for short lengths
constexpr int HIST_SMEM = 4096;
__global__ void k_len_hist(int64_t nrows, const int64_t* __restrict__ ptr, int64_t nbins,
                           unsigned long long* __restrict__ hist) {
  __shared__ unsigned int sh[HIST_SMEM];
  const int64_t local = nbins < HIST_SMEM ? nbins : HIST_SMEM;
  for (int b = threadIdx.x; b < local; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  GRID_STRIDE(i, nrows) {
    const int64_t L = ptr[i + 1] - ptr[i];
    if (L < HIST_SMEM) atomicAdd(sh + L, 1u);
    else atomicAdd(hist + L, 1ull);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < local; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, (unsigned long long)sh[b]);
}

// hyb_split_width (formats.py:364-370): sorted(lens)[ceil(2n/3) - 1] from the
// histogram's cumulative counts
static int64_t hyb_width(const RowView& v, int64_t maxlen, cudaStream_t s) {
  const int64_t n = v.nrows;
  if (n == 0) return 0;
  const int64_t nbins = maxlen + 1;
  Buf h = alloc(nbins * 8, s);
  SVB_CUDA_TRY(cudaMemsetAsync(h->ptr, 0, nbins * 8, s));
  k_len_hist<<<grid_for(n, 256, 4), 256, 0, s>>>(n, ptr<int64_t>(v.ptr), nbins,
                                                ptr<unsigned long long>(h));
  SVB_CHECK_LAUNCH();
  std::vector<unsigned long long> hh(nbins);
  SVB_CUDA_TRY(cudaMemcpyAsync(hh.data(), h->ptr, nbins * 8, cudaMemcpyDeviceToHost, s));
  SVB_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t need = (2 * n + 2) / 3;  // ceil(2n/3)
  int64_t cum = 0;
  for (int64_t L = 0; L < nbins; ++L) {
    cum += (int64_t)hh[L];
    if (cum >= need) return L;
  }
  return maxlen;
}

// ---------------------------------------------------------------------------
// builders
// ---------------------------------------------------------------------------
// ELL(width) cells from the first min(len, width) entries of every row;
// column-major, sentinel col = ncols / value 0 (formats.py:339-348, 379-385)
__global__ void k_to_ell(int64_t nrows, int64_t ncols, int64_t width, const int64_t* __restrict__ ptr,
                         const int* __restrict__ cols, const double* __restrict__ vals,
                         int* __restrict__ ecols, double* __restrict__ evals) {
  GRID_STRIDE(i, nrows) {
    const int64_t s = ptr[i], len = ptr[i + 1] - s;
    for (int64_t k = 0; k < width; ++k) {
      const bool has = k < len;
      ecols[k * nrows + i] = has ? cols[s + k] : (int)ncols;
      evals[k * nrows + i] = has ? vals[s + k] : 0.0;
    }
  }
}

__global__ void k_spill_count(int64_t nrows, int64_t width, const int64_t* __restrict__ ptr,
                              int64_t* __restrict__ cnt) {
  GRID_STRIDE(i, nrows) { const int64_t d = ptr[i + 1] - ptr[i] - width; cnt[i] = d > 0 ? d : 0; }
}

__global__ void k_spill_fill(int64_t nrows, int64_t width, const int64_t* __restrict__ ptr,
                             const int* __restrict__ cols, const double* __restrict__ vals,
                             const int64_t* __restrict__ sptr, int* __restrict__ srows,
                             int* __restrict__ scols, double* __restrict__ svals) {
  GRID_STRIDE(i, nrows) {
    int64_t o = sptr[i];
    for (int64_t k = ptr[i] + width; k < ptr[i + 1]; ++k, ++o) {
      srows[o] = (int)i;
      scols[o] = cols[k];
      svals[o] = vals[k];
    }
  }
}

// diagonal occupancy bitmap: bit (col - row + nrows - 1); test before the
// atomic so the hot diagonals of banded matrices are not contended
// diagonal-occupancy bitmap over row tiles staged in shared memory (coalesced
// col_idx reads); a bit is only atomically set when it is still clear
constexpr int TILE_ROWS = 256;
__global__ void __launch_bounds__(TILE_ROWS) k_diag_bits(int64_t nrows, const int64_t* __restrict__ ptr,
                                                         const int* __restrict__ cols, unsigned* __restrict__ bits) {
  constexpr int CAP = 8192;
  constexpr int LONG = 64;   // longer rows are marked by a warp (power-law tails)
  __shared__ int scol[CAP];
  __shared__ long long dcache[DIAG_CACHE];
  __shared__ int lrows[TILE_ROWS];
  __shared__ int nl;
  diag_cache_init(dcache);
  if (threadIdx.x == 0) nl = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (nrows + TILE_ROWS - 1) / TILE_ROWS;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const StagedRows<int64_t> t = stage_row_tile<int64_t, TILE_ROWS, CAP>(tile, nrows, ptr, cols, scol);
    auto col = [&](int64_t k) { return t.staged ? scol[k] : __ldg(cols + t.base + k); };
    const int64_t i = t.r0 + threadIdx.x;
    if (i < t.r1) {
      const int64_t s0 = ptr[i] - t.base, e = ptr[i + 1] - t.base;
      if (e - s0 > LONG) {
        lrows[atomicAdd(&nl, 1)] = threadIdx.x;
      } else {
        for (int64_t k = s0; k < e; ++k) mark_diag(bits, (long long)col(k) - i + nrows - 1, dcache);
      }
    }
    __syncthreads();
    for (int q = warp; q < nl; q += TILE_ROWS / 32) {
      const int64_t r = t.r0 + lrows[q];
      for (int64_t k = ptr[r] - t.base + lane, e = ptr[r + 1] - t.base; k < e; k += 32)
        mark_diag(bits, (long long)col(k) - r + nrows - 1, dcache);
    }
    __syncthreads();   // every warp is done with nl / lrows
    if (threadIdx.x == 0) nl = 0;
  }
}

__global__ void k_popc(int64_t nwords, const unsigned* __restrict__ bits, int64_t* __restrict__ cnt) {
  GRID_STRIDE(w, nwords) cnt[w] = __popc(bits[w]);
}

__global__ void k_bits_to_offsets(int64_t nwords, int64_t nrows, const unsigned* __restrict__ bits,
                                  const int64_t* __restrict__ pos, long long* __restrict__ offs) {
  GRID_STRIDE(w, nwords) {
    unsigned b = bits[w];
    int64_t o = pos[w];
    while (b) {
      const int t = __ffs(b) - 1;
      offs[o++] = w * 32 + t - (nrows - 1);
      b &= b - 1;
    }
  }
}

constexpr int DIA_CAP = 4096;  // DIA_OFFSET_CAP (formats.py:18)

// DIA data, every cell written once (no memset): thread-per-row over row
// tiles that the TMA engine bulk-copies (cols, vals and the row-pointer
// slice) into a shared-memory ring, DIA_NS tiles in flight per CTA; the
// entry bounds of the tiles to issue are prefetched DIA_PF tiles ahead
// with cp.async.  (Round 1 staged each tile with one synchronous load per
// thread: ncu 42 % of DRAM bandwidth, 208 us at config 2.)  The row's
// (strictly increasing) columns are merged against the ascending offsets,
// so data[d*n + i] is the value at column i + off[d] or 0.  Consecutive
// threads write consecutive rows of each diagonal: coalesced stores.
constexpr int DIA_R = 256, DIA_TILE_CAP = 2560, DIA_NS = 3, DIA_PF = 4, DIA_BR = 8;
__global__ void __launch_bounds__(DIA_R) k_csr_to_dia(int64_t nrows, int64_t ndiag, const long long* __restrict__ offs,
                                                     const int64_t* __restrict__ ptr, const int* __restrict__ cols,
                                                     const double* __restrict__ vals, double* __restrict__ data) {
  using Lay = RingLayout<int64_t, DIA_R, DIA_TILE_CAP, true>;
  extern __shared__ __align__(128) unsigned char dsm[];
  long long* so = reinterpret_cast<long long*>(dsm + DIA_NS * Lay::STAGE);
  __shared__ alignas(8) uint64_t bar[DIA_NS];
  __shared__ RingDesc desc[DIA_NS];
  __shared__ alignas(16) int64_t bnd[DIA_BR][2];
  const int tid = threadIdx.x;
  for (int k = tid; k < ndiag; k += blockDim.x) so[k] = offs[k];
  const int64_t ntiles = (nrows + DIA_R - 1) / DIA_R;
  const uint64_t policy = l2_evict_first_policy();
  auto issue = [&](int st, int64_t tile, int64_t e0, int64_t e1) {
    const int64_t r0 = tile * DIA_R, r1 = min(r0 + DIA_R, nrows);
    ring_issue<int64_t, DIA_R, DIA_TILE_CAP, true>(dsm + st * Lay::STAGE, &bar[st], &desc[st], r0, r1, e0, e1, ptr,
                                                   cols, vals, policy);
  };
  auto prefetch = [&](int64_t local) {
    const int64_t tile = blockIdx.x + local * gridDim.x;
    if (tile < ntiles) {
      const int sl = (int)(local % DIA_BR);
      cp_async_small<8>(&bnd[sl][0], ptr + tile * DIA_R);
      cp_async_small<8>(&bnd[sl][1], ptr + min(tile * DIA_R + DIA_R, nrows));
    }
    cp_async_commit();
  };
  if (tid == 0) {
    for (int st = 0; st < DIA_NS; ++st) mbar_init(&bar[st], 1);
    for (int st = 0; st < DIA_NS; ++st) {
      const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
      if (tile < ntiles) issue(st, tile, ptr[tile * DIA_R], ptr[min(tile * DIA_R + DIA_R, nrows)]);
    }
    for (int k = 0; k < DIA_PF; ++k) prefetch(DIA_NS + k);
  }
  __syncthreads();
  for (int64_t tile = blockIdx.x, it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = (int)(it % DIA_NS);
    const int64_t tn = tile + (int64_t)DIA_NS * gridDim.x;
    if (tid == 0) prefetch(it + DIA_NS + DIA_PF);
    mbar_wait(&bar[st], (uint32_t)(it / DIA_NS) & 1u);
    const RingDesc d = desc[st];
    const unsigned char* stage = dsm + st * Lay::STAGE;
    const double* sval = reinterpret_cast<const double*>(stage) + d.voff;
    const int* scol = reinterpret_cast<const int*>(stage + Lay::SV) + d.coff;
    const int64_t* sp = reinterpret_cast<const int64_t*>(stage + Lay::SV + Lay::SC) + d.poff;
    const int64_t nst = d.staged;
    const int64_t i = d.r0 + tid;
    if (i < d.r1) {
      int64_t k = sp[tid] - d.e0;
      const int64_t e = sp[tid + 1] - d.e0;
      const bool sm = e <= nst;   // the whole row is staged
      auto col = [&](int64_t q) { return sm ? scol[q] : __ldg(cols + d.e0 + q); };
      auto val = [&](int64_t q) { return sm ? sval[q] : __ldg(vals + d.e0 + q); };
      int c = k < e ? col(k) : 0;
      for (int64_t g = 0; g < ndiag; ++g) {
        double v = 0.0;
        if (k < e && (long long)c - i == so[g]) {
          v = val(k);
          ++k;
          if (k < e) c = col(k);
        }
        data[g * nrows + i] = v;
      }
    }
    __syncthreads();   // stage st is free again
    if (tid == 0 && tn < ntiles) {
      cp_async_wait<DIA_PF>();
      const int sl = (int)((it + DIA_NS) % DIA_BR);
      fence_proxy_async_smem();
      issue(st, tn, bnd[sl][0], bnd[sl][1]);
    }
  }
  cp_async_wait<0>();
}

static svb_matrix* new_like(const RowView& v, int fmt) {
  auto m = new svb_matrix();
  m->fmt = fmt;
  m->nrows = v.nrows;
  m->ncols = v.ncols;
  m->nnz = v.nnz;
  return m;
}

static svb_matrix* build_csr(const RowView& v, cudaStream_t s) {
  auto m = new_like(v, SVB_CSR);
  m->ptr64 = want_ptr64(v.nnz);
  if (m->ptr64) m->ptr = v.ptr;
  else {
    m->ptr = alloc((v.nrows + 1) * 4, s);
    narrow_i64_to_i32(ptr<int64_t>(v.ptr), ptr<int32_t>(m->ptr), v.nrows + 1, s);
  }
  m->cols = v.cols;
  m->vals = v.vals;
  return m;
}

static svb_matrix* build_coo(const RowView& v, const svb_matrix* src, cudaStream_t s) {
  auto m = new_like(v, SVB_COO);
  m->ptr64 = want_ptr64(v.nnz);
  if (v.rows) m->rows = v.rows;
  else {
    svb_matrix tmp;  // CSR-shaped view over the row pointer for the expansion kernel
    tmp.nrows = v.nrows;
    tmp.nnz = v.nnz;
    tmp.ptr64 = true;
    tmp.ptr = v.ptr;
    m->rows = ptr_to_rows(&tmp, s);
  }
  m->cols = v.cols;
  m->vals = v.vals;
  (void)src;
  return m;
}

static svb_matrix* build_ell(const RowView& v, int64_t max_cells, cudaStream_t s) {
  const int64_t width = v.nnz ? max_row_len(v, s) : 0;
  if (max_cells > 0 && width > 0 && width > max_cells / std::max<int64_t>(v.nrows, 1))
    throw Error{SVB_INAPPLICABLE, "ELL would need " + std::to_string(v.nrows) + " x " +
                                      std::to_string(width) + " cells, above the device cap of " +
                                      std::to_string(max_cells) + "; ELL is inapplicable"};
  auto m = new_like(v, SVB_ELL);
  m->width = width;
  m->cols = alloc(width * v.nrows * 4, s);
  m->vals = alloc(width * v.nrows * 8, s);
  if (width) {
    k_to_ell<<<grid_for(v.nrows, 256), 256, 0, s>>>(v.nrows, v.ncols, width, ptr<int64_t>(v.ptr),
                                                    ptr<int>(v.cols), ptr<double>(v.vals), ptr<int>(m->cols),
                                                    ptr<double>(m->vals));
    SVB_CHECK_LAUNCH();
  }
  return m;
}

// DiaMatrix keeps no nnz; report the stored (in-range) cells like svb_dia_create
static int64_t dia_stored(const std::vector<int64_t>& offs, int64_t nrows, int64_t ncols) {
  int64_t stored = 0;
  for (const int64_t off : offs) {
    const int64_t lo = off < 0 ? -off : 0, hi = std::min<int64_t>(nrows, ncols - off);
    if (hi > lo) stored += hi - lo;
  }
  return stored;
}

// DIA data from the row view, every cell written once (m->offs on device)
static void fill_dia(const RowView& v, svb_matrix* m, cudaStream_t s) {
  using Lay = RingLayout<int64_t, DIA_R, DIA_TILE_CAP, true>;
  const size_t dsm = DIA_NS * Lay::STAGE + (size_t)m->ndiag * 8;
  static const bool attr = [] {   // once per process (thread-safe static init)
    SVB_CUDA_TRY(cudaFuncSetAttribute(k_csr_to_dia, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(DIA_NS * Lay::STAGE + (size_t)DIA_CAP * 8)));
    return true;
  }();
  (void)attr;
  int per = 0;
  SVB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_csr_to_dia, DIA_R, dsm));
  const int64_t ntiles = (v.nrows + DIA_R - 1) / DIA_R;
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count() * std::max(per, 1)));
  k_csr_to_dia<<<g, DIA_R, dsm, s>>>(v.nrows, m->ndiag, ptr<long long>(m->offs), ptr<int64_t>(v.ptr),
                                     ptr<int>(v.cols), ptr<double>(v.vals), ptr<double>(m->vals));
  SVB_CHECK_LAUNCH();
}

static svb_matrix* build_dia(const RowView& v, const svb_matrix* src, cudaStream_t s) {
  const int64_t nbits = v.nrows + v.ncols - 1;
  const int64_t nwords = (nbits + 31) / 32;
  Buf bits;
  std::vector<int64_t> cached;   // sorted offsets the feature pass left on the CSR handle
  bool have_offs = false;
  if (src->fmt == SVB_CSR) {   // the bitmap feature extraction left on the handle
    std::lock_guard<std::mutex> lk(src->mu);
    if (src->diag_bits && src->diag_bits->bytes >= (size_t)nwords * 4) {
      bits = src->diag_bits;
      if (src->diag_offs_valid) {
        cached = src->diag_offs;
        have_offs = true;
      }
    }
  }
  if (have_offs) {
    const int64_t ndiag = (int64_t)cached.size();
    auto m = new_like(v, SVB_DIA);
    m->ndiag = ndiag;
    m->offs = alloc(ndiag * 8, s);
    m->vals = alloc(ndiag * v.nrows * 8, s);
    m->h_offs = cached;
    if (ndiag) {
      SVB_CUDA_TRY(cudaMemcpyAsync(m->offs->ptr, m->h_offs.data(), ndiag * 8, cudaMemcpyHostToDevice, s));
      fill_dia(v, m, s);
    }
    m->nnz = dia_stored(m->h_offs, v.nrows, v.ncols);
    return m;
  }
  const bool reused = (bool)bits;
  if (!reused) {
    bits = alloc(nwords * 4, s);
    SVB_CUDA_TRY(cudaMemsetAsync(bits->ptr, 0, nwords * 4, s));
  }
  if (v.nnz && !reused) {
    k_diag_bits<<<grid_for(v.nrows, TILE_ROWS), TILE_ROWS, 0, s>>>(v.nrows, ptr<int64_t>(v.ptr), ptr<int>(v.cols),
                                                       ptr<unsigned>(bits));
    SVB_CHECK_LAUNCH();
  }
  Buf cnt = alloc(nwords * 8, s);
  k_popc<<<grid_for(nwords, 256), 256, 0, s>>>(nwords, ptr<unsigned>(bits), ptr<int64_t>(cnt));
  SVB_CHECK_LAUNCH();
  Buf pos = alloc((nwords + 1) * 8, s);
  const int64_t ndiag = exclusive_scan_total(ptr<int64_t>(cnt), ptr<int64_t>(pos), nwords, s);
  if (ndiag > DIA_CAP)
    throw Error{SVB_INAPPLICABLE, "matrix populates " + std::to_string(ndiag) +
                                      " diagonals, above the cap of " + std::to_string(DIA_CAP) +
                                      "; DIA is inapplicable"};
  auto m = new_like(v, SVB_DIA);
  m->ndiag = ndiag;
  m->offs = alloc(ndiag * 8, s);
  m->vals = alloc(ndiag * v.nrows * 8, s);
  if (ndiag) {
    k_bits_to_offsets<<<grid_for(nwords, 256), 256, 0, s>>>(nwords, v.nrows, ptr<unsigned>(bits),
                                                            ptr<int64_t>(pos), ptr<long long>(m->offs));
    SVB_CHECK_LAUNCH();
    fill_dia(v, m, s);
    m->h_offs.resize(ndiag);
    SVB_CUDA_TRY(cudaMemcpyAsync(m->h_offs.data(), m->offs->ptr, ndiag * 8, cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
  }
  m->nnz = dia_stored(m->h_offs, v.nrows, v.ncols);
  return m;
}

static svb_matrix* build_hyb(const RowView& v, cudaStream_t s) {
  const int64_t maxlen = v.nnz ? max_row_len(v, s) : 0;
  const int64_t w = hyb_width(v, maxlen, s);
  auto m = new_like(v, SVB_HYB);
  m->width = w;
  m->cols = alloc(w * v.nrows * 4, s);
  m->vals = alloc(w * v.nrows * 8, s);
  const unsigned g = grid_for(v.nrows, 256);
  if (w) {
    k_to_ell<<<g, 256, 0, s>>>(v.nrows, v.ncols, w, ptr<int64_t>(v.ptr), ptr<int>(v.cols),
                               ptr<double>(v.vals), ptr<int>(m->cols), ptr<double>(m->vals));
    SVB_CHECK_LAUNCH();
  }
  Buf cnt = alloc(v.nrows * 8, s);
  k_spill_count<<<g, 256, 0, s>>>(v.nrows, w, ptr<int64_t>(v.ptr), ptr<int64_t>(cnt));
  SVB_CHECK_LAUNCH();
  m->ptr = alloc((v.nrows + 1) * 8, s);
  m->spill_nnz = exclusive_scan_total(ptr<int64_t>(cnt), ptr<int64_t>(m->ptr), v.nrows, s);
  m->rows = alloc(m->spill_nnz * 4, s);
  m->scols = alloc(m->spill_nnz * 4, s);
  m->svals = alloc(m->spill_nnz * 8, s);
  if (m->spill_nnz) {
    k_spill_fill<<<g, 256, 0, s>>>(v.nrows, w, ptr<int64_t>(v.ptr), ptr<int>(v.cols), ptr<double>(v.vals),
                                   ptr<int64_t>(m->ptr), ptr<int>(m->rows), ptr<int>(m->scols),
                                   ptr<double>(m->svals));
    SVB_CHECK_LAUNCH();
  }
  return m;
}

}  // namespace svb

using namespace svb;

extern "C" {

int svb_convert(const svb_matrix* src, int target, int64_t max_ell_cells, void* stream,
                svb_matrix** out) {
  return guard([&] {
    SVB_REQUIRE(src && out, SVB_INVALID, "null handle");
    SVB_REQUIRE(target >= SVB_COO && target <= SVB_HYB, SVB_INVALID, "unknown format tag");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    RowView v = row_view(src, s);
    svb_matrix* m = nullptr;
    switch (target) {
      case SVB_COO: m = build_coo(v, src, s); break;
      case SVB_CSR: m = build_csr(v, s); break;
      case SVB_ELL: m = build_ell(v, max_ell_cells, s); break;
      case SVB_DIA: m = build_dia(v, src, s); break;
      default: m = build_hyb(v, s); break;
    }
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(m);
  });
}

int svb_hyb_split_width(const svb_matrix* m, void* stream, int64_t* width_out) {
  return guard([&] {
    SVB_REQUIRE(m && width_out, SVB_INVALID, "null handle");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    RowView v = row_view(m, s);
    *width_out = hyb_width(v, v.nnz ? max_row_len(v, s) : 0, s);
  });
}

}  // extern "C"
