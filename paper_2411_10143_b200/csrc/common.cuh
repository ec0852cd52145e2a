// Shared device/host plumbing for libspmvtune_b200 (sm_100a).
//
// Status codes, the thread-local error string behind svb_last_error(), the
// stream-ordered device allocator wrapper, grid sizing for the 148-SM B200,
// and the fp summation-order primitives every "exact" kernel uses
// (numpy's pairwise sum).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>

#include "../../include/spmvtune_b200.h"

namespace svb {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
const char* get_error();

struct Error {
  int code;
  std::string msg;
};

#define SVB_CUDA_TRY(expr)                                                   \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      throw ::svb::Error{_e == cudaErrorMemoryAllocation ? SVB_OOM : SVB_CUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    }                                                                        \
  } while (0)

// Every launch of one of this library's kernels is counted (svb_launch_count):
// bench.py reports the count for its timed region as evidence that the
// native path ran.
void note_launches(int64_t n);
#define SVB_CHECK_LAUNCH()                 \
  do {                                     \
    ::svb::note_launches(1);               \
    SVB_CUDA_TRY(cudaGetLastError());      \
  } while (0)

#define SVB_REQUIRE(cond, code, msg)                \
  do {                                                \
    if (!(cond)) throw ::svb::Error{(code), (msg)};   \
  } while (0)

// Runs `body` and maps exceptions onto status codes (never throws across
// the C ABI).
template <class F>
int guard(F&& body) {
  try {
    body();
    return SVB_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return SVB_OOM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SVB_INVALID;
  }
}

// Row pointers are int32 on the device unless nnz >= 2^31 (config 5 on one
// GPU).  SPMVTUNE_FORCE_PTR64=1 makes every new CSR/COO handle use int64 row
// pointers regardless of size: the test hook that runs the int64 kernels on
// small matrices the CPU oracle can check.
inline bool want_ptr64(int64_t nnz) {
  static const bool forced = [] {
    const char* e = std::getenv("SPMVTUNE_FORCE_PTR64");
    return e && e[0] == '1';
  }();
  return forced || nnz >= INT32_MAX;
}

// ---------------------------------------------------------------------------
// device memory: stream-ordered pool allocations, shared between immutable
// matrix handles (a CSR->COO conversion shares col/val buffers, for example)
// ---------------------------------------------------------------------------
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = 0;  // freed stream-ordered on the allocating stream
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
};
using Buf = std::shared_ptr<DevBuf>;

Buf alloc(size_t bytes, cudaStream_t s);

template <class T>
inline T* ptr(const Buf& b) {
  return b ? static_cast<T*>(b->ptr) : nullptr;
}

int sm_count();

// Grid for a grid-stride streaming kernel: enough CTAs to cover the work,
// capped at `per_sm` resident CTAs on every SM.
inline unsigned grid_for(int64_t work_items, int block, int per_sm = 8) {
  int64_t need = (work_items + block - 1) / block;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (need < 1) need = 1;
  return (unsigned)(need < cap ? need : cap);
}

// ---------------------------------------------------------------------------
// summation-order primitives (numpy pairwise sum)
// ---------------------------------------------------------------------------
// numpy pairwise leaf (n <= 128): 8 strided accumulators, fixed combine tree,
// sequential tail.  `get(i)` yields the i-th addend.
template <class T, class G>
__device__ __forceinline__ T pw_leaf(const G& get, int64_t lo, int64_t n) {
  if (n < 8) {
    T r = T(-0.0);
    for (int64_t i = 0; i < n; ++i) r = r + get(lo + i);
    return r;
  }
  T r0 = get(lo + 0), r1 = get(lo + 1), r2 = get(lo + 2), r3 = get(lo + 3);
  T r4 = get(lo + 4), r5 = get(lo + 5), r6 = get(lo + 6), r7 = get(lo + 7);
  const int64_t lim = n - (n % 8);
  int64_t i = 8;
  for (; i < lim; i += 8) {
    r0 = r0 + get(lo + i + 0);
    r1 = r1 + get(lo + i + 1);
    r2 = r2 + get(lo + i + 2);
    r3 = r3 + get(lo + i + 3);
    r4 = r4 + get(lo + i + 4);
    r5 = r5 + get(lo + i + 5);
    r6 = r6 + get(lo + i + 6);
    r7 = r7 + get(lo + i + 7);
  }
  T res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res = res + get(lo + i);
  return res;
}

// numpy's pairwise recursion with a caller-supplied evaluator `leaf(lo, n)` for the
// nodes of at most `span` addends (span >= 128; the split rule is numpy's at
// every level): used to enumerate the leaves of a long segment and later to
// combine leaf sums computed in parallel by a warp, in identical order, and
// to walk the top of very long segments in warp-sized subtrees.
template <class T, class L>
__device__ T pw_traverse(const L& leaf, int64_t lo, int64_t n, int64_t span = 128) {
  if (n <= span) return leaf(lo, n);
  struct Frame {
    int64_t lo, n;
    T left;
    int state;
  };
  Frame st[28];
  int sp = 0;
  st[0] = {lo, n, T(0), 0};
  T ret = T(0);
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= span) {
      ret = leaf(f.lo, f.n);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.lo, n2, T(0), 0};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.lo + n2, f.n - n2, T(0), 0};
      ++sp;
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

// Full numpy pairwise sum: n <= 128 is a leaf, otherwise split at
// n2 = n/2 rounded down to a multiple of 8 and add the halves.  The
// recursion is unrolled onto an explicit stack (depth <= 28 covers 2^31
// addends) so the common short-segment path carries no call frames.
template <class T, class G>
__device__ T pw_sum(const G& get, int64_t lo, int64_t n) {
  if (n <= 128) return pw_leaf<T>(get, lo, n);
  struct Frame {
    int64_t lo, n;
    T left;
    int state;
  };
  Frame st[28];
  int sp = 0;
  st[0] = {lo, n, T(0), 0};
  T ret = T(0);
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pw_leaf<T>(get, f.lo, f.n);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.lo, n2, T(0), 0};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.lo + n2, f.n - n2, T(0), 0};
      ++sp;
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

// One np.add.reduceat segment [s, e), e > s: p[s] + pairwise(p[s+1:e]).
template <class T, class G>
__device__ __forceinline__ T segment_sum(const G& get, int64_t s, int64_t e) {
  T head = get(s);
  if (e - s == 1) return head;
  return head + pw_sum<T>(get, s + 1, e - s - 1);
}

// ---------------------------------------------------------------------------
// cache-hinted loads: streamed matrix arrays bypass L1 allocation, the
// gathered x vector uses the read-only path and stays cached
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ long long ld_stream(const long long* p) {
  long long v;
  asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <class T>
__device__ __forceinline__ T ld_x(const T* p) {
  return __ldg(p);
}

// ---------------------------------------------------------------------------
// 1-D bulk copies (TMA engine, no tensor map) into shared memory, completed
// on an mbarrier: one elected thread arms the barrier with the byte count and
// issues the copies; every thread waits on the phase parity.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// the same with an L2 eviction-priority hint (createpolicy): streamed matrix
// arrays are marked evict-first so the gathered x vector stays L2-resident
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// small asynchronous global -> shared copies (LDGSTS): the issuing thread
// does not stall on them; commit groups and wait for all but the newest N
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* dst, const void* src) {
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// order earlier generic-proxy accesses of shared memory before later bulk
// copies into it (buffer reuse)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace svb
