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
template <class G>
__device__ __forceinline__ void warp_row_runs(const G& col, int64_t s, int64_t e, int64_t diag0,
                                              unsigned* __restrict__ bits, long long* dcache,
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
    if (valid) mark_diag(bits, (long long)c + diag0, dcache);
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

template <class P, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_features(int64_t nrows, const P* __restrict__ ptr,
                                                    const int* __restrict__ cols,
                                                    unsigned* __restrict__ bits, FeatAcc* out) {
  constexpr int CAP = 8192;  // staged column indices per tile (32 KB)
  __shared__ int scol[CAP];
  __shared__ long long dcache[DIAG_CACHE];
  __shared__ int lrows[BLOCK];
  __shared__ int nl;
  diag_cache_init(dcache);   // (the tile loop's first __syncthreads orders it)
  if (threadIdx.x == 0) nl = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FeatAcc a{0, 0, 0, 0, 0, LLONG_MAX};
  const int64_t ntiles = (nrows + BLOCK - 1) / BLOCK;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const StagedRows<P> t = stage_row_tile<P, BLOCK, CAP>(tile, nrows, ptr, cols, scol);
    auto col = [&](int64_t k) { return t.staged ? scol[k] : __ldg(cols + t.base + k); };
    const int64_t i = t.r0 + threadIdx.x;
    if (i < t.r1) {
      const int64_t s = (int64_t)ptr[i] - t.base, e = (int64_t)ptr[i + 1] - t.base, L = e - s;
      a.sum_r += (unsigned long long)L;
      a.sum_r2 += (unsigned long long)(L * L);
      a.max_r = max(a.max_r, (long long)L);
      a.min_r = min(a.min_r, (long long)L);
      if (L > FEAT_LONG) {
        lrows[atomicAdd(&nl, 1)] = threadIdx.x;
      } else if (L > 0) {
        const int64_t diag0 = nrows - 1 - i;
        const int c0 = col(s);
        int prev = c0;
        int64_t run = 1, best = 1;
        for (int64_t k = s;;) {
          mark_diag(bits, (long long)prev + diag0, dcache);
          if (++k >= e) break;
          const int c = col(k);
          run = (c == prev + 1) ? run + 1 : 1;
          best = max(best, run);
          prev = c;
        }
        a.span += (unsigned long long)(prev - c0);
        a.runs += (unsigned long long)best;
      }
    }
    __syncthreads();
    for (int q = warp; q < nl; q += BLOCK / 32) {
      const int64_t r = t.r0 + lrows[q];
      const int64_t s = (int64_t)ptr[r] - t.base, e = (int64_t)ptr[r + 1] - t.base;
      long long best, span;
      warp_row_runs(col, s, e, nrows - 1 - r, bits, dcache, &best, &span);
      if (lane == 0) {
        a.span += (unsigned long long)span;
        a.runs += (unsigned long long)best;
      }
    }
    __syncthreads();   // every warp is done with nl / lrows
    if (threadIdx.x == 0) nl = 0;
  }
  block_reduce_store<BLOCK>(a, out);
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
__global__ void k_bits_to_offsets(int64_t nwords, const unsigned* __restrict__ bits, int64_t base,
                                  long long* __restrict__ out, int64_t cap, unsigned long long* __restrict__ cnt) {
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

extern "C" int svb_features(const svb_matrix* m, int64_t* agg, void* stream) {
  return guard([&] {
    SVB_REQUIRE(m && agg, SVB_INVALID, "null handle");
    SVB_REQUIRE(m->fmt == SVB_CSR, SVB_UNSUPPORTED_CONFIG, "extract_features expects CSR");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nbits = m->nrows + m->ncols - 1;
    const int64_t nwords = (nbits + 31) / 32;
    Buf bits = alloc(nwords * 4, s);
    Buf acc = alloc(sizeof(FeatAcc) + 8, s);
    SVB_CUDA_TRY(cudaMemsetAsync(bits->ptr, 0, nwords * 4, s));
    FeatAcc init{0, 0, 0, 0, 0, LLONG_MAX};
    SVB_CUDA_TRY(cudaMemcpyAsync(acc->ptr, &init, sizeof(FeatAcc), cudaMemcpyHostToDevice, s));
    SVB_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(acc->ptr) + sizeof(FeatAcc), 0, 8, s));
    constexpr int B = 256;
    const unsigned g = grid_for(m->nrows, B, 8);
    if (m->ptr64)
      k_features<long long, B><<<g, B, 0, s>>>(m->nrows, ptr<long long>(m->ptr), ptr<int>(m->cols),
                                              ptr<unsigned>(bits), ptr<FeatAcc>(acc));
    else
      k_features<int, B><<<g, B, 0, s>>>(m->nrows, ptr<int>(m->ptr), ptr<int>(m->cols),
                                        ptr<unsigned>(bits), ptr<FeatAcc>(acc));
    SVB_CHECK_LAUNCH();
    auto* ndiag_d = reinterpret_cast<unsigned long long*>(static_cast<char*>(acc->ptr) + sizeof(FeatAcc));
    k_popcount<<<grid_for(nwords, 256, 4), 256, 0, s>>>(nwords, ptr<unsigned>(bits), ndiag_d);
    SVB_CHECK_LAUNCH();
    struct {
      FeatAcc a;
      unsigned long long ndiag;
    } h;
    SVB_CUDA_TRY(cudaMemcpyAsync(&h, acc->ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    {  // complete now: kept for a later DIA conversion of this handle
      detach(bits);
      std::lock_guard<std::mutex> lk(m->mu);
      m->diag_bits = bits;
    }
    agg[0] = (int64_t)h.a.sum_r;
    agg[1] = (int64_t)h.a.sum_r2;
    agg[2] = h.a.max_r;
    agg[3] = m->nrows ? h.a.min_r : 0;
    agg[4] = (int64_t)h.a.span;
    agg[5] = (int64_t)h.a.runs;
    agg[6] = (int64_t)h.ndiag;
  });
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
