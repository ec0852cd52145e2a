// Structural features on the device: extract_features (features.py:68-156).
//
// The fifteen reference features are float formulas over seven exact
// integer aggregates.  One fused pass over row_ptr and
// col_idx produces six of them (row-length sum / square-sum / max / min,
// row span sum, longest-consecutive-run sum) and sets the diagonal-occupancy
// bitmap; a popcount pass yields the seventh (ndiag).  Integer arithmetic
// makes the aggregates independent of the reduction order, and the host
// evaluates the floats with the reference's own expressions, so the feature
// vector is bit-identical to the CPU path.
#include <algorithm>
#include <climits>
#include <cstddef>
#include <mutex>
#include <vector>

#include "matrix.cuh"

namespace svb {

struct FeatAcc {
  unsigned long long sum_r, sum_r2, span, runs;
  long long max_r, min_r;
};

template <int BLOCK>
__device__ void block_reduce_store(FeatAcc a, FeatAcc* out) {
  __shared__ FeatAcc sh[BLOCK / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a.sum_r += __shfl_xor_sync(0xffffffffu, a.sum_r, o);
    a.sum_r2 += __shfl_xor_sync(0xffffffffu, a.sum_r2, o);
    a.span += __shfl_xor_sync(0xffffffffu, a.span, o);
    a.runs += __shfl_xor_sync(0xffffffffu, a.runs, o);
    a.max_r = max(a.max_r, (long long)__shfl_xor_sync(0xffffffffu, a.max_r, o));
    a.min_r = min(a.min_r, (long long)__shfl_xor_sync(0xffffffffu, a.min_r, o));
  }
  if (lane == 0) sh[wid] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    FeatAcc t = sh[0];
    for (int w = 1; w < BLOCK / 32; ++w) {
      t.sum_r += sh[w].sum_r;
      t.sum_r2 += sh[w].sum_r2;
      t.span += sh[w].span;
      t.runs += sh[w].runs;
      t.max_r = max(t.max_r, sh[w].max_r);
      t.min_r = min(t.min_r, sh[w].min_r);
    }
    atomicAdd(&out->sum_r, t.sum_r);
    atomicAdd(&out->sum_r2, t.sum_r2);
    atomicAdd(&out->span, t.span);
    atomicAdd(&out->runs, t.runs);
    atomicMax(&out->max_r, t.max_r);
    atomicMin(&out->min_r, t.min_r);
  }
}

// Rows longer than FEAT_LONG entries are handed to a warp: one thread
// walking a power-law row of thousands of entries (a dependent bitmap probe
// per entry) would otherwise set the kernel time on its own.
constexpr int FEAT_LONG = 64;

// Longest run of consecutive columns and the diagonal marks of one row by a
// warp, in the sequential recurrence's terms (run = c == prev + 1 ? run + 1
// : 1, best = max run); returns (best, last - first column) on every lane.
template <class D, class G>
__device__ __forceinline__ void warp_row_runs(const G& col, int64_t s, int64_t e, D diag0,
                                              unsigned* __restrict__ bits, D* dcache,
                                              long long* best_out, long long* span_out) {
  const int lane = threadIdx.x & 31;
  long long best = 0, carry = 0;   // run length through the previous chunk's last entry
  int prev_last = 0;
  const int first = col(s);
  int last = first;
  for (int64_t base = s; base < e; base += 32) {
    const int64_t k = base + lane;
    const bool valid = k < e;
    const int c = valid ? col(k) : 0;
    int pc = __shfl_up_sync(0xffffffffu, c, 1);
    if (lane == 0) pc = prev_last;
    const bool brk = valid && ((k == s) || c != pc + 1);
    if (valid) mark_diag(bits, (D)c + diag0, dcache);
    const unsigned B = __ballot_sync(0xffffffffu, brk);
    const unsigned upto = B & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
    long long run = 0;
    if (valid) run = upto ? (long long)(lane - (31 - __clz(upto)) + 1) : carry + lane + 1;
    long long m = run;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, (long long)__shfl_xor_sync(0xffffffffu, m, o));
    best = max(best, m);
    const int nv = (int)(e - base < 32 ? e - base : 32);
    carry = __shfl_sync(0xffffffffu, run, nv - 1);
    prev_last = __shfl_sync(0xffffffffu, c, nv - 1);
    last = prev_last;
  }
  *best_out = best;
  *span_out = (long long)last - first;
}

struct FeatOut {
  FeatAcc a;
  unsigned long long ndiag;                  // popcount of the bitmap
  unsigned long long rows_read, cols_read;   // row_ptr / col_idx elements consumed
  unsigned long long noffs;                  // offsets written below (may exceed the cap)
  unsigned long long nxl;                    // rows handed to k_features_xl
  int cancelled;
  int pad;
  long long offs[4096];                      // diagonal offsets (unordered) when ndiag <= 4096
};

// Rows longer than FEAT_XL entries (power-law hubs: thousands of entries)
// leave the tile pipeline: walked by one warp inside a tile they held the
// whole CTA at its next barrier for a global round trip per 32 columns
// (0.61 ms for a 1 M-row power-law matrix; 0.35 ms with this path).  The
// tile pass lists them (row, begin, end) and k_features_xl walks each with
// a whole CTA: every warp summarises a contiguous part of the row (first and
// last column, longest run inside, run length from its start and at its
// end, whether it is one run), and the parts are joined left to right — the
// run lengths of the sequential recurrence.
constexpr int FEAT_XL = 2048;

struct RunPart {
  long long first, last, best, pre, suf, len;
  bool full;
};
__device__ __forceinline__ RunPart join_parts(const RunPart& a, const RunPart& b) {
  if (a.len == 0) return b;
  if (b.len == 0) return a;
  const bool link = b.first == a.last + 1;
  RunPart c;
  c.first = a.first;
  c.last = b.last;
  c.best = max(max(a.best, b.best), link ? a.suf + b.pre : 0ll);
  c.pre = (a.full && link) ? a.len + b.pre : a.pre;
  c.suf = (b.full && link) ? b.len + a.suf : b.suf;
  c.full = a.full && b.full && link;
  c.len = a.len + b.len;
  return c;
}

// one warp: columns [s, e) of a row (s < e), diagonal marks included
template <class D>
__device__ RunPart warp_part(const int* __restrict__ cols, int64_t s, int64_t e, D diag0, unsigned* __restrict__ bits,
                             D* dcache) {
  const int lane = threadIdx.x & 31;
  RunPart r{0, 0, 0, 0, 0, e - s, true};
  long long carry = 0, pre = -1;
  int prev_last = 0;
  for (int64_t base = s; base < e; base += 32) {
    const int64_t k = base + lane;
    const bool valid = k < e;
    const int c = valid ? __ldg(cols + k) : 0;
    int pc = __shfl_up_sync(0xffffffffu, c, 1);
    if (lane == 0) pc = prev_last;
    const bool brk = valid && ((k == s) || c != pc + 1);
    if (valid) mark_diag(bits, (D)c + diag0, dcache);
    const unsigned B = __ballot_sync(0xffffffffu, brk);
    const unsigned upto = B & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
    long long run = 0;
    if (valid) run = upto ? (long long)(lane - (31 - __clz(upto)) + 1) : carry + lane + 1;
    long long m = run;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, (long long)__shfl_xor_sync(0xffffffffu, m, o));
    r.best = max(r.best, m);
    // the first break after the part's first entry ends the leading run
    const unsigned later = base == s ? (B & ~1u) : B;
    if (pre < 0 && later) pre = base - s + (__ffs(later) - 1);
    if (base == s) r.first = __shfl_sync(0xffffffffu, c, 0);
    const int nv = (int)(e - base < 32 ? e - base : 32);
    carry = __shfl_sync(0xffffffffu, run, nv - 1);
    prev_last = __shfl_sync(0xffffffffu, c, nv - 1);
  }
  r.last = prev_last;
  r.suf = carry;
  r.full = pre < 0;
  r.pre = pre < 0 ? r.len : pre;
  return r;
}

struct XlRow {
  long long row, beg, end;
};

template <class D>
__global__ void __launch_bounds__(256) k_features_xl(int64_t nrows, const int* __restrict__ cols,
                                                     unsigned* __restrict__ bits, const XlRow* __restrict__ list,
                                                     FeatOut* out, const volatile int* cancel) {
  __shared__ D dcache[DIAG_CACHE];
  __shared__ RunPart parts[8];
  __shared__ int stop;
  diag_cache_init(dcache);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long count = out->nxl;
  for (unsigned long long q = blockIdx.x; q < count; q += gridDim.x) {
    if (threadIdx.x == 0) stop = cancel ? *cancel : 0;   // one reading per CTA: a uniform exit
    __syncthreads();
    if (stop) return;
    const XlRow xr = list[q];
    const int64_t len = xr.end - xr.beg, per = (len + 7) / 8;
    const int64_t a = xr.beg + min((int64_t)warp * per, len), b = xr.beg + min((int64_t)(warp + 1) * per, len);
    RunPart p{0, 0, 0, 0, 0, 0, true};
    if (a < b) p = warp_part<D>(cols, a, b, (D)(nrows - 1 - xr.row), bits, dcache);
    if (lane == 0) parts[warp] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
      RunPart t = parts[0];
      for (int w = 1; w < 8; ++w) t = join_parts(t, parts[w]);
      atomicAdd(&out->a.span, (unsigned long long)(t.last - t.first));
      atomicAdd(&out->a.runs, (unsigned long long)t.best);
    }
    __syncthreads();
  }
}

// One pass over row_ptr and col_idx through the row-tile ring (matrix.cuh):
// one thread per row walks its staged columns (run lengths, span, diagonal
// marks) in 32-bit arithmetic (ncu, round 1 kernel: 65 instructions per
// entry, issue-bound at 0.2 of HBM); rows longer than FEAT_LONG go to a
// warp, rows longer than FEAT_XL to k_features_xl.  A tile's entries are staged up to the stage capacity (a row that
// crosses the end reads global memory).  Thread 0 keeps the row-pointer
// bounds of the tiles it will issue FEAT_PF tiles ahead with cp.async, so
// no refill waits on a dependent row_ptr load.  Thread 0 polls the cancel
// flag one tile ahead and, once it is raised, stops refilling the ring; the
// tiles already in flight are drained without being walked.  The flag is a
// device word (an L2 read per tile): svb_features_cancel raises it with a
// 4-byte copy on a side stream, which the copy engine performs while the
// kernel runs.  (Polling host-mapped memory instead costs a PCIe round trip
// per tile, and those reads serialise: 12 ms for a 4 M-row pass.)  Rows and
// entries actually walked are counted (the reference's TraversalCounter,
// features.py:60-65).
constexpr int FEAT_R = 256, FEAT_CAP = 5120, FEAT_NS = 3, FEAT_PF = 4, FEAT_BR = 8;


template <class P, class D>
__global__ void __launch_bounds__(FEAT_R) k_features(int64_t nrows, const P* __restrict__ ptr,
                                                     const int* __restrict__ cols, unsigned* __restrict__ bits,
                                                     FeatOut* out, const volatile int* cancel,
                                                     XlRow* __restrict__ xl) {
  using Lay = RingLayout<P, FEAT_R, FEAT_CAP, false>;
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ alignas(8) uint64_t bar[FEAT_NS];
  __shared__ RingDesc desc[FEAT_NS];
  __shared__ D dcache[DIAG_CACHE];
  __shared__ int lrows[FEAT_R];
  __shared__ alignas(16) P bnd[FEAT_BR][2];   // entry bounds of prefetched tiles
  __shared__ int nlong[2], sstop;   // long-row count, double-buffered by iteration parity
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  diag_cache_init(dcache);
  const int64_t ntiles = (nrows + FEAT_R - 1) / FEAT_R;
  const uint64_t policy = l2_evict_first_policy();
  int cflag = 0;   // thread 0: the cancel flag as read one tile ago
  auto issue = [&](int st, int64_t tile, int64_t e0, int64_t e1) {
    const int64_t r0 = tile * FEAT_R, r1 = min(r0 + FEAT_R, nrows);
    ring_issue<P, FEAT_R, FEAT_CAP, false>(ring + st * Lay::STAGE, &bar[st], &desc[st], r0, r1, e0, e1, ptr, cols,
                                          nullptr, policy);
  };
  auto prefetch = [&](int64_t local) {   // bounds of this CTA's local-th tile -> bnd (thread 0)
    const int64_t tile = blockIdx.x + local * gridDim.x;
    if (tile < ntiles) {
      const int sl = (int)(local % FEAT_BR);
      cp_async_small<sizeof(P)>(&bnd[sl][0], ptr + tile * FEAT_R);
      cp_async_small<sizeof(P)>(&bnd[sl][1], ptr + min(tile * FEAT_R + FEAT_R, nrows));
    }
    cp_async_commit();   // one group per call, empty or not: wait_group counts them
  };
  if (tid == 0) {
    nlong[0] = nlong[1] = 0;
    sstop = 0;
    for (int st = 0; st < FEAT_NS; ++st) mbar_init(&bar[st], 1);
    if (cancel) cflag = *cancel;
    for (int st = 0; st < FEAT_NS; ++st) {
      const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
      if (tile < ntiles && !cflag)
        issue(st, tile, (int64_t)ptr[tile * FEAT_R], (int64_t)ptr[min(tile * FEAT_R + FEAT_R, nrows)]);
    }
    if (cflag) sstop = 1;
    for (int k = 0; k < FEAT_PF; ++k) prefetch(FEAT_NS + k);
  }
  __syncthreads();
  FeatAcc a{0, 0, 0, 0, 0, LLONG_MAX};
  unsigned long long rows_read = 0, cols_read = 0;
  int64_t stop_at = sstop ? -1 : INT64_MAX;   // first iteration whose tile was not issued
  for (int64_t tile = blockIdx.x, it = 0; tile < ntiles && it < stop_at; tile += gridDim.x, ++it) {
    const int st = (int)(it % FEAT_NS);
    int& nl = nlong[it & 1];
    int nxt_cancel = 0;
    const int64_t tn = tile + (int64_t)FEAT_NS * gridDim.x;   // the tile this stage takes next
    if (tid == 0) {
      nlong[(it + 1) & 1] = 0;   // last read before the previous iteration's final barrier
      if (cancel) nxt_cancel = *cancel;   // consumed after this tile (latency hidden)
      prefetch(it + FEAT_NS + FEAT_PF);
    }
    mbar_wait(&bar[st], (uint32_t)(it / FEAT_NS) & 1u);
    const RingDesc d = desc[st];
    const bool walk = stop_at == INT64_MAX;
    const unsigned char* stage = ring + st * Lay::STAGE;
    const int* scol = reinterpret_cast<const int*>(stage + Lay::SV) + d.coff;
    const P* sp = reinterpret_cast<const P*>(stage + Lay::SV + Lay::SC) + d.poff;
    const int64_t nst = d.staged;
    auto col = [&](int64_t k) { return k < nst ? scol[k] : __ldg(cols + d.e0 + k); };
    const int64_t i = d.r0 + tid;
    if (walk && i < d.r1) {
      const int64_t s = (int64_t)sp[tid] - d.e0, e = (int64_t)sp[tid + 1] - d.e0, L = e - s;
      a.sum_r += (unsigned long long)L;
      a.sum_r2 += (unsigned long long)(L * L);
      a.max_r = max(a.max_r, (long long)L);
      a.min_r = min(a.min_r, (long long)L);
      if (L > FEAT_XL) {
        const unsigned long long q = atomicAdd(&out->nxl, 1ull);
        xl[q] = XlRow{(long long)i, (long long)(sp[tid]), (long long)(sp[tid + 1])};
      } else if (L > FEAT_LONG) {
        lrows[atomicAdd(&nl, 1)] = tid;
      } else if (L > 0) {
        // 32-bit walk over the row's columns (shared memory when the whole
        // row is staged)
        const int* rp = e <= nst ? scol + s : cols + d.e0 + s;
        const int n = (int)L;
        const D dg = (D)(nrows - 1 - i);
        const int c0 = rp[0];
        int prev = c0, run = 1, best = 1;
        mark_diag(bits, (D)c0 + dg, dcache);
        for (int k = 1; k < n; ++k) {
          const int c = rp[k];
          run = (c == prev + 1) ? run + 1 : 1;
          best = max(best, run);
          mark_diag(bits, (D)c + dg, dcache);
          prev = c;
        }
        a.span += (unsigned long long)((long long)prev - c0);
        a.runs += (unsigned long long)best;
      }
    }
    if (walk && tid == 0) {
      rows_read += (unsigned long long)(d.r1 - d.r0 + 1);
      cols_read += (unsigned long long)(d.e1 - d.e0);
    }
    __syncthreads();
    for (int q = warp; q < nl; q += FEAT_R / 32) {
      const int64_t r = d.r0 + lrows[q];
      const int64_t s = (int64_t)sp[lrows[q]] - d.e0, e = (int64_t)sp[lrows[q] + 1] - d.e0;
      long long best, span;
      warp_row_runs(col, s, e, (D)(nrows - 1 - r), bits, dcache, &best, &span);
      if (lane == 0) {
        a.span += (unsigned long long)span;
        a.runs += (unsigned long long)best;
      }
    }
    if (tid == 0) {
      if (cflag) sstop = 1;   // raised one tile ago: stop refilling from here
      cflag = nxt_cancel;
    }
    __syncthreads();   // stage st, nl/lrows and sstop settled
    if (sstop && stop_at == INT64_MAX) stop_at = it + FEAT_NS;   // drain what is in flight
    if (tid == 0) {
      if (!sstop && tn < ntiles) {
        cp_async_wait<FEAT_PF>();   // this tile's bounds (prefetched FEAT_PF tiles ago) landed
        const int sl = (int)((it + FEAT_NS) % FEAT_BR);
        const int64_t e0 = (int64_t)bnd[sl][0], e1 = (int64_t)bnd[sl][1];
        fence_proxy_async_smem();
        issue(st, tn, e0, e1);
      }
    }
  }
  cp_async_wait<0>();
  block_reduce_store<FEAT_R>(a, &out->a);
  if (tid == 0) {
    if (rows_read) atomicAdd(&out->rows_read, rows_read);
    if (cols_read) atomicAdd(&out->cols_read, cols_read);
    if (sstop) atomicExch(&out->cancelled, 1);
  }
}

__global__ void k_popcount(int64_t nwords, const unsigned* __restrict__ bits,
                           unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x)
    c += __popc(bits[w]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ unsigned long long sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    atomicAdd(out, t);
  }
}

// set bits of the diagonal bitmap -> offsets (bit - (nrows - 1) + shift),
// unordered (the host sorts them)
// (skip_above: the popcount; above the cap the list is not wanted and the
// counter atomics of millions of set words would be pure contention)
__global__ void k_bits_to_offsets(int64_t nwords, const unsigned* __restrict__ bits, int64_t base,
                                  long long* __restrict__ out, int64_t cap, unsigned long long* __restrict__ cnt,
                                  const unsigned long long* __restrict__ skip_above = nullptr) {
  if (skip_above && *skip_above > (unsigned long long)cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = *skip_above;
    return;
  }
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    unsigned b = bits[w];
    if (!b) continue;
    unsigned long long at = atomicAdd(cnt, (unsigned long long)__popc(b));
    while (b) {
      const int k = __ffs(b) - 1;
      b &= b - 1;
      if ((int64_t)at < cap) out[at] = (long long)(w * 32 + k) + base;
      ++at;
    }
  }
}

}  // namespace svb

using namespace svb;

// ---------------------------------------------------------------------------
// Feature jobs: the pass is enqueued (svb_features_start) and its result
// block (aggregates, traversal counters, cancel outcome and the diagonal
// offsets) lands in pinned host memory behind an event, so the caller never
// blocks inside the library while the pass runs: it polls, may raise the
// cancel flag (a device word the kernel reads one tile ahead), and
// collects the result with svb_features_finish.  A completed, uncancelled
// pass leaves its diagonal bitmap and sorted offsets on the CSR handle for
// a later DIA conversion (no second pass over col_idx, no offset scan).
// ---------------------------------------------------------------------------
struct svb_features_job {
  const svb_matrix* m = nullptr;
  cudaStream_t s = nullptr;
  FeatOut* host = nullptr;     // pinned result block
  int* flag = nullptr;         // device cancel word; 0 whenever the job is idle
  cudaEvent_t done = nullptr;
  bool cancel_requested = false;
  Buf bits, out, xl;
};

namespace {
std::mutex g_job_mu;
std::vector<svb_features_job*> g_job_pool;   // pinned blocks are slow to allocate: recycle jobs

// the side stream and the pinned source word of cancel requests
struct CancelPath {
  cudaStream_t s = nullptr;
  int* one = nullptr;
  CancelPath() {
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaHostAlloc((void**)&one, sizeof(int), cudaHostAllocDefault) != cudaSuccess)
      throw Error{SVB_CUDA, "cannot create the feature-cancel stream"};
    *one = 1;
  }
};
CancelPath& cancel_path() {
  static CancelPath p;
  return p;
}

svb_features_job* job_get() {
  {
    std::lock_guard<std::mutex> lk(g_job_mu);
    if (!g_job_pool.empty()) {
      auto* j = g_job_pool.back();
      g_job_pool.pop_back();
      return j;
    }
  }
  auto* j = new svb_features_job();
  try {
    SVB_CUDA_TRY(cudaHostAlloc((void**)&j->host, sizeof(FeatOut), cudaHostAllocDefault));
    SVB_CUDA_TRY(cudaMalloc((void**)&j->flag, 16));
    SVB_CUDA_TRY(cudaMemset(j->flag, 0, 16));
    SVB_CUDA_TRY(cudaEventCreateWithFlags(&j->done, cudaEventDisableTiming));
  } catch (...) {
    if (j->host) cudaFreeHost(j->host);
    if (j->flag) cudaFree(j->flag);
    delete j;
    throw;
  }
  return j;
}

void job_put(svb_features_job* j) {
  j->bits.reset();
  j->out.reset();
  j->xl.reset();
  j->m = nullptr;
  j->cancel_requested = false;
  std::lock_guard<std::mutex> lk(g_job_mu);
  g_job_pool.push_back(j);
}
}  // namespace

extern "C" int svb_features_start(const svb_matrix* m, int precancelled, void* stream, svb_features_job** job) {
  return guard([&] {
    SVB_REQUIRE(m && job, SVB_INVALID, "null handle");
    SVB_REQUIRE(m->fmt == SVB_CSR, SVB_UNSUPPORTED_CONFIG, "extract_features expects CSR");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    svb_features_job* j = job_get();
    try {
      j->m = m;
      j->s = s;
      j->cancel_requested = precancelled != 0;
      cancel_path();   // created before the first job can be cancelled
      const int64_t nbits = m->nrows + m->ncols - 1;
      const int64_t nwords = (nbits + 31) / 32;
      j->bits = alloc(nwords * 4, s);
      j->out = alloc(sizeof(FeatOut), s);
      j->xl = alloc((m->nnz / (FEAT_XL + 1) + 1) * sizeof(XlRow), s);   // rows longer than FEAT_XL
      auto* out = ptr<FeatOut>(j->out);
      SVB_CUDA_TRY(cudaMemsetAsync(j->bits->ptr, 0, nwords * 4, s));
      SVB_CUDA_TRY(cudaMemsetAsync(out, 0, offsetof(FeatOut, offs), s));
      const long long big = LLONG_MAX;
      SVB_CUDA_TRY(cudaMemcpyAsync(&out->a.min_r, &big, 8, cudaMemcpyHostToDevice, s));
      const int64_t ntiles = (m->nrows + FEAT_R - 1) / FEAT_R;
      if (precancelled) {   // nothing is read: report the cancellation only
        const int one = 1;
        SVB_CUDA_TRY(cudaMemcpyAsync(&out->cancelled, &one, 4, cudaMemcpyHostToDevice, s));
      } else if (ntiles > 0) {
        const size_t dsm32 = FEAT_NS * RingLayout<int, FEAT_R, FEAT_CAP, false>::STAGE;
        const size_t dsm64 = FEAT_NS * RingLayout<long long, FEAT_R, FEAT_CAP, false>::STAGE;
        static const bool attr = [&] {
          SVB_CUDA_TRY(cudaFuncSetAttribute(k_features<int, unsigned>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)dsm32));
          SVB_CUDA_TRY(cudaFuncSetAttribute(k_features<int, long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)dsm32));
          SVB_CUDA_TRY(cudaFuncSetAttribute(k_features<long long, unsigned>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm64));
          SVB_CUDA_TRY(cudaFuncSetAttribute(k_features<long long, long long>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm64));
          return true;
        }();
        (void)attr;
        const unsigned g = (unsigned)std::min<int64_t>(ntiles, (int64_t)sm_count() * 3);
        // 32-bit diagonal indices whenever they fit (nrows + ncols - 1 < 2^32)
        const bool narrow = nbits < (int64_t(1) << 32);
        auto* bitsp = ptr<unsigned>(j->bits);
        if (m->ptr64) {
          if (narrow)
            k_features<long long, unsigned><<<g, FEAT_R, dsm64, s>>>(m->nrows, ptr<long long>(m->ptr), ptr<int>(m->cols),
                                                                     bitsp, out, j->flag, ptr<XlRow>(j->xl));
          else
            k_features<long long, long long><<<g, FEAT_R, dsm64, s>>>(m->nrows, ptr<long long>(m->ptr),
                                                                      ptr<int>(m->cols), bitsp, out, j->flag,
                                                                      ptr<XlRow>(j->xl));
        } else {
          if (narrow)
            k_features<int, unsigned><<<g, FEAT_R, dsm32, s>>>(m->nrows, ptr<int>(m->ptr), ptr<int>(m->cols), bitsp,
                                                               out, j->flag, ptr<XlRow>(j->xl));
          else
            k_features<int, long long><<<g, FEAT_R, dsm32, s>>>(m->nrows, ptr<int>(m->ptr), ptr<int>(m->cols), bitsp,
                                                                out, j->flag, ptr<XlRow>(j->xl));
        }
        SVB_CHECK_LAUNCH();
        if (m->nnz > FEAT_XL) {   // the listed extra-long rows, a CTA each
          const unsigned gx = (unsigned)std::min<int64_t>(m->nnz / (FEAT_XL + 1) + 1, (int64_t)sm_count() * 4);
          if (narrow)
            k_features_xl<unsigned><<<gx, 256, 0, s>>>(m->nrows, ptr<int>(m->cols), bitsp, ptr<XlRow>(j->xl), out,
                                                        j->flag);
          else
            k_features_xl<long long><<<gx, 256, 0, s>>>(m->nrows, ptr<int>(m->cols), bitsp, ptr<XlRow>(j->xl), out,
                                                         j->flag);
          SVB_CHECK_LAUNCH();
        }
      }
      k_popcount<<<grid_for(nwords, 256, 4), 256, 0, s>>>(nwords, ptr<unsigned>(j->bits), &out->ndiag);
      SVB_CHECK_LAUNCH();
      k_bits_to_offsets<<<grid_for(nwords, 256, 4), 256, 0, s>>>(nwords, ptr<unsigned>(j->bits), -(m->nrows - 1),
                                                                out->offs, 4096, &out->noffs, &out->ndiag);
      SVB_CHECK_LAUNCH();
      SVB_CUDA_TRY(cudaMemcpyAsync(j->host, out, offsetof(FeatOut, offs), cudaMemcpyDeviceToHost, s));
      // the offsets only when they fit the DIA cap (a second copy ordered after the first)
      SVB_CUDA_TRY(cudaMemcpyAsync(j->host->offs, out->offs, sizeof(out->offs), cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaEventRecord(j->done, s));
    } catch (...) {
      cudaStreamSynchronize(s);
      job_put(j);
      throw;
    }
    *job = j;
  });
}

extern "C" int svb_features_cancel(svb_features_job* job) {
  return guard([&] {
    SVB_REQUIRE(job, SVB_INVALID, "null job");
    if (job->cancel_requested) return;
    job->cancel_requested = true;
    CancelPath& c = cancel_path();
    SVB_CUDA_TRY(cudaMemcpyAsync(job->flag, c.one, sizeof(int), cudaMemcpyHostToDevice, c.s));
  });
}

extern "C" int svb_features_query(svb_features_job* job, int* done) {
  return guard([&] {
    SVB_REQUIRE(job && done, SVB_INVALID, "null job");
    const cudaError_t e = cudaEventQuery(job->done);
    if (e == cudaErrorNotReady) {
      *done = 0;
      return;
    }
    SVB_CUDA_TRY(e);
    *done = 1;
  });
}

extern "C" int svb_features_wait(svb_features_job* job) {
  return guard([&] {
    SVB_REQUIRE(job, SVB_INVALID, "null job");
    SVB_CUDA_TRY(cudaEventSynchronize(job->done));
  });
}

extern "C" int svb_features_finish(svb_features_job* job, int64_t* agg, int64_t* counters, int* cancelled) {
  return guard([&] {
    SVB_REQUIRE(job, SVB_INVALID, "null job");
    struct Put {   // the job goes back to the pool whatever happens below
      svb_features_job* j;
      ~Put() { job_put(j); }
    } put{job};
    SVB_CUDA_TRY(cudaEventSynchronize(job->done));
    if (job->cancel_requested) {   // re-arm the flag before the job is reused
      CancelPath& c = cancel_path();
      SVB_CUDA_TRY(cudaMemsetAsync(job->flag, 0, sizeof(int), c.s));
      SVB_CUDA_TRY(cudaStreamSynchronize(c.s));
    }
    const FeatOut& h = *job->host;
    const svb_matrix* m = job->m;
    if (counters) {
      counters[0] = (int64_t)h.rows_read;
      counters[1] = (int64_t)h.cols_read;
    }
    const int was_cancelled = h.cancelled || job->cancel_requested;
    if (cancelled) *cancelled = was_cancelled;
    if (agg) {
      agg[0] = (int64_t)h.a.sum_r;
      agg[1] = (int64_t)h.a.sum_r2;
      agg[2] = h.a.max_r;
      agg[3] = m->nrows ? h.a.min_r : 0;
      agg[4] = (int64_t)h.a.span;
      agg[5] = (int64_t)h.a.runs;
      agg[6] = (int64_t)h.ndiag;
    }
    if (!h.cancelled) {   // complete: kept for a later DIA conversion of this handle
      detach(job->bits);
      std::lock_guard<std::mutex> lk(m->mu);
      m->diag_bits = job->bits;
      m->diag_offs.clear();
      m->diag_offs_valid = h.noffs <= 4096;
      if (m->diag_offs_valid) {
        m->diag_offs.assign(h.offs, h.offs + h.noffs);
        std::sort(m->diag_offs.begin(), m->diag_offs.end());
      }
    }
  });
}

extern "C" int svb_features(const svb_matrix* m, int64_t* agg, void* stream) {
  svb_features_job* job = nullptr;
  const int st = svb_features_start(m, 0, stream, &job);
  if (st != SVB_OK) return st;
  return svb_features_finish(job, agg, nullptr, nullptr);
}

extern "C" int svb_diag_offsets(const svb_matrix* m, int64_t shift, int64_t* out_host, int64_t cap, int64_t* count,
                                void* stream) {
  return guard([&] {
    SVB_REQUIRE(m && count && (cap == 0 || out_host), SVB_INVALID, "null argument");
    SVB_REQUIRE(m->fmt == SVB_CSR, SVB_UNSUPPORTED_CONFIG, "diagonal offsets need a CSR matrix");
    Buf bits;
    {
      std::lock_guard<std::mutex> lk(m->mu);
      bits = m->diag_bits;
    }
    if (!bits) {   // the feature pass builds (and caches) the bitmap
      int64_t agg[7];
      const int st = svb_features(m, agg, stream);
      if (st != SVB_OK) throw Error{st, get_error()};
      std::lock_guard<std::mutex> lk(m->mu);
      bits = m->diag_bits;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nwords = (m->nrows + m->ncols - 1 + 31) / 32;
    Buf tmp = alloc(8 + std::max<int64_t>(cap, 1) * 8, s);
    auto* cnt = ptr<unsigned long long>(tmp);
    SVB_CUDA_TRY(cudaMemsetAsync(cnt, 0, 8, s));
    k_bits_to_offsets<<<grid_for(nwords, 256, 4), 256, 0, s>>>(nwords, ptr<unsigned>(bits), shift - (m->nrows - 1),
                                                              ptr<long long>(tmp) + 1, cap, cnt);
    SVB_CHECK_LAUNCH();
    unsigned long long c = 0;
    SVB_CUDA_TRY(cudaMemcpyAsync(&c, cnt, 8, cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *count = (int64_t)c;
    const int64_t k = std::min<int64_t>((int64_t)c, cap);
    if (k > 0) {
      SVB_CUDA_TRY(cudaMemcpyAsync(out_host, ptr<long long>(tmp) + 1, k * 8, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
      std::sort(out_host, out_host + k);
    }
  });
}
