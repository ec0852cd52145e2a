// Library plumbing and the container half of the C ABI:
// svb_{coo,csr,ell,dia,hyb}_create, svb_matrix_{destroy,info_get,download}.
// Mirrors the reference containers (formats.py:50-260); host-side validation
// with the reference's error messages lives in the Python layer.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <climits>
#include <cstring>
#include <atomic>
#include <mutex>
#include <thread>

#include <vector>

#include "matrix.cuh"

namespace svb {

// ---------------------------------------------------------------------------
// errors / allocation / device facts
// ---------------------------------------------------------------------------
static thread_local std::string tls_error;
void set_error(const std::string& msg) { tls_error = msg; }
const char* get_error() { return tls_error.c_str(); }

static std::atomic<int64_t> g_launches{0};
void note_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

DevBuf::~DevBuf() {
  if (ptr) cudaFreeAsync(ptr, stream);
}

Buf alloc(size_t bytes, cudaStream_t s) {
  auto b = std::make_shared<DevBuf>();
  b->bytes = bytes;
  b->stream = s;
  if (bytes) {
    // +128 B tail: bulk (TMA) copies round their byte counts up to 16 B
    cudaError_t e = cudaMallocAsync(&b->ptr, bytes + 128, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error{e == cudaErrorMemoryAllocation ? SVB_OOM : SVB_CUDA,
                  std::string("device allocation of ") + std::to_string(bytes) +
                      " bytes failed: " + cudaGetErrorString(e)};
    }
  }
  return b;
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
  }
  return cached;
}

Buf upload(const void* host, size_t bytes, cudaStream_t s) {
  Buf b = alloc(bytes, s);
  if (bytes) SVB_CUDA_TRY(cudaMemcpyAsync(b->ptr, host, bytes, cudaMemcpyHostToDevice, s));
  return b;
}

// ---------------------------------------------------------------------------
// index width conversion kernels
// ---------------------------------------------------------------------------
__global__ void k_narrow(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (int32_t)src[i];
}
__global__ void k_widen(const int32_t* __restrict__ src, int64_t* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_to_f32(const double* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

// rows [r0, r0 + n) of a row pointer, rebased to start at 0
template <class Pin, class Pout>
__global__ void k_rebase_ptr(const Pin* __restrict__ src, Pout* __restrict__ dst, int64_t n1) {
  const int64_t base = (int64_t)src[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (Pout)((int64_t)src[i] - base);
}

void narrow_i64_to_i32(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  k_narrow<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
  SVB_CHECK_LAUNCH();
}
void widen_i32_to_i64(const int32_t* src, int64_t* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  k_widen<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
  SVB_CHECK_LAUNCH();
}
void ptr_to_i64(const svb_matrix* m, int64_t* dst, cudaStream_t s) {
  if (m->ptr64)
    SVB_CUDA_TRY(cudaMemcpyAsync(dst, m->ptr->ptr, (m->nrows + 1) * 8, cudaMemcpyDeviceToDevice, s));
  else
    widen_i32_to_i64(ptr<int32_t>(m->ptr), dst, m->nrows + 1, s);
}

static Buf to_f32(const Buf& src, int64_t n, cudaStream_t s) {
  Buf out = alloc(n * sizeof(float), s);
  if (n > 0) {
    k_to_f32<<<grid_for(n, 256), 256, 0, s>>>(ptr<double>(src), ptr<float>(out), n);
    SVB_CHECK_LAUNCH();
  }
  return out;
}

const float* vals_f32(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (!m->vals32) {
    int64_t n = m->vals ? (int64_t)(m->vals->bytes / 8) : 0;
    m->vals32 = to_f32(m->vals, n, s);
    detach(m->vals32);
  }
  return ptr<float>(m->vals32);
}
const float* svals_f32(const svb_matrix* m, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (!m->svals32) {
    m->svals32 = to_f32(m->svals, m->spill_nnz, s);
    detach(m->svals32);
  }
  return ptr<float>(m->svals32);
}

int64_t exclusive_scan_total(const int64_t* counts, int64_t* out, int64_t n, cudaStream_t s) {
  // out[0..n] = exclusive prefix of counts[0..n-1] with the total at out[n]
  SVB_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
  if (n > 0) {
    size_t tmp_bytes = 0;
    SVB_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, counts, out + 1, n, s));
    Buf tmp = alloc(tmp_bytes, s);
    SVB_CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp->ptr, tmp_bytes, counts, out + 1, n, s));
  }
  int64_t total = 0;
  SVB_CUDA_TRY(cudaMemcpyAsync(&total, out + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SVB_CUDA_TRY(cudaStreamSynchronize(s));
  return total;
}

// row_ptr from sorted COO rows: ptr[i] = lower_bound(rows, i) (formats.py:327-330)
template <class P>
__global__ void k_rows_to_ptr(const int32_t* __restrict__ rows, int64_t nnz, int64_t nrows,
                              P* __restrict__ ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (rows[mid] < i) lo = mid + 1; else hi = mid;
    }
    ptr[i] = (P)lo;
  }
}

Buf rows_to_ptr(const int32_t* rows, int64_t nnz, int64_t nrows, bool ptr64, cudaStream_t s) {
  Buf p = alloc((nrows + 1) * (ptr64 ? 8 : 4), s);
  if (ptr64)
    k_rows_to_ptr<long long><<<grid_for(nrows + 1, 256), 256, 0, s>>>(rows, nnz, nrows, ptr<long long>(p));
  else
    k_rows_to_ptr<int32_t><<<grid_for(nrows + 1, 256), 256, 0, s>>>(rows, nnz, nrows, ptr<int32_t>(p));
  SVB_CHECK_LAUNCH();
  return p;
}

// rows from a CSR row pointer (formats.py:285-287): one thread per row
template <class P>
__global__ void k_ptr_to_rows(const P* __restrict__ ptr, int64_t nrows, int32_t* __restrict__ rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = ptr[i], e = ptr[i + 1];
    for (int64_t k = s; k < e; ++k) rows[k] = (int32_t)i;
  }
}

Buf ptr_to_rows(const svb_matrix* m, cudaStream_t s) {
  Buf r = alloc(m->nnz * 4, s);
  if (m->nnz > 0) {
    if (m->ptr64)
      k_ptr_to_rows<long long><<<grid_for(m->nrows, 128), 128, 0, s>>>(ptr<long long>(m->ptr), m->nrows, ptr<int32_t>(r));
    else
      k_ptr_to_rows<int32_t><<<grid_for(m->nrows, 128), 128, 0, s>>>(ptr<int32_t>(m->ptr), m->nrows, ptr<int32_t>(r));
    SVB_CHECK_LAUNCH();
  }
  return r;
}


// ---------------------------------------------------------------------------
// host slabs of a row-partitioned rank (distributed_solve_slab)
// ---------------------------------------------------------------------------
// min / max of the column indices (atomics on one pair per CTA)
template <class C>
__global__ void k_col_minmax(const C* __restrict__ c, int64_t n, long long* __restrict__ mm) {
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = (long long)c[i];
    lo = v < lo ? v : lo;
    hi = v > hi ? v : hi;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, (long long)__shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, (long long)__shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

// global -> window-relative int32 columns (in place when C is int32)
template <class C>
__global__ void k_cols_rebase(const C* __restrict__ src, int32_t* __restrict__ dst, int64_t n, int64_t shift) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (int32_t)((int64_t)src[i] - shift);
}

// CsrMatrix structure rules (formats.py:113-138) on the device: flags[0]
// row_ptr decreasing, flags[1] columns not strictly increasing in a row
template <class P>
__global__ void k_csr_check(int64_t nrows, const P* __restrict__ ptr, const int32_t* __restrict__ cols,
                            int* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = (int64_t)ptr[i], e = (int64_t)ptr[i + 1];
    if (e < s) {
      flags[0] = 1;
      continue;
    }
    for (int64_t k = s + 1; k < e; ++k)
      if (cols[k] <= cols[k - 1]) {
        flags[1] = 1;
        break;
      }
  }
}

// window-relative int32 columns -> global int32 (export)
__global__ void k_cols_shift(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n, int64_t shift) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (int32_t)((int64_t)src[i] + shift);
}

}  // namespace svb

using namespace svb;

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Device -> pageable host copies of 12 MB and more through a pinned staging
// buffer drained by several host threads, part by part as each part's DMA
// completes.  The driver's own pageable path stages through one thread:
// a 16 MB solve vector came down in 0.91 ms, staged 0.68 ms (32 MB: 1.66 ->
// 1.26; profiles/pageable_copy.py).  The same staging for host -> device
// (threads filling the buffer, each issuing its part's DMA) measured SLOWER
// than the driver's path (16 MB 1.58 vs 0.85 ms: fresh threads initialising
// the runtime for their cudaMemcpyAsync), so uploads copy directly.  Same
// semantics as cudaMemcpy from pageable memory: stream-ordered, and the
// call returns when the host buffer may be reused (H2D) / holds the data.
namespace {
constexpr int64_t STAGE_MIN = 12 << 20;      // below: plain cudaMemcpyAsync (8 MB staged: 0.50 vs 0.43 ms)
constexpr int64_t STAGE_MAX = 64ll << 20;    // staging buffer (pinned, portable)
std::mutex g_stage_mu;
char* g_stage = nullptr;
int64_t g_stage_bytes = 0;

char* stage_buffer(int64_t want) {
  if (g_stage_bytes < want) {
    if (g_stage) SVB_CUDA_TRY(cudaFreeHost(g_stage));
    g_stage = nullptr;
    g_stage_bytes = 0;
    void* p = nullptr;
    SVB_CUDA_TRY(cudaHostAlloc(&p, want, cudaHostAllocPortable));
    g_stage = static_cast<char*>(p);
    g_stage_bytes = want;
  }
  return g_stage;
}

int stage_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(8u, hw ? hw / 2 : 1u));
}
}  // namespace

static void require_index_range(int64_t nrows, int64_t ncols) {
  SVB_REQUIRE(nrows >= 1 && ncols >= 1, SVB_DIM_MISMATCH, "matrix dimensions must be positive");
  SVB_REQUIRE(nrows < INT32_MAX && ncols < INT32_MAX, SVB_INAPPLICABLE,
              "dimensions >= 2^31 are not supported by the int32 device index layout");
}

static Buf upload_i32(const int64_t* host, int64_t n, cudaStream_t s) {
  Buf out = alloc(n * 4, s);
  if (n > 0) {
    Buf stage = upload(host, n * 8, s);
    narrow_i64_to_i32(ptr<int64_t>(stage), ptr<int32_t>(out), n, s);
  }
  return out;
}

extern "C" {

const char* svb_last_error(void) { return get_error(); }
int svb_launch_count(int64_t* out) {
  *out = g_launches.load();
  return SVB_OK;
}
int svb_abi_version(void) { return SVB_ABI_VERSION; }

int svb_init(int device) {
  return guard([&] {
    SVB_CUDA_TRY(cudaSetDevice(device));
    // keep freed pool memory cached: conversions and workspaces recycle it
    cudaMemPool_t pool;
    SVB_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    SVB_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    sm_count();
  });
}

int svb_stream_sync(void* stream) {
  return guard([&] { SVB_CUDA_TRY(cudaStreamSynchronize(S(stream))); });
}

int svb_stream_create(int priority, void** out) {
  return guard([&] {
    int lo = 0, hi = 0;
    SVB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // priority > 0 asks for the highest (solver), < 0 for the lowest (advisor)
    const int p = priority > 0 ? hi : (priority < 0 ? lo : 0);
    cudaStream_t s;
    SVB_CUDA_TRY(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, p));
    *out = s;
  });
}
int svb_stream_destroy(void* stream) {
  return guard([&] { SVB_CUDA_TRY(cudaStreamDestroy(S(stream))); });
}
// CUDA graphs: a host loop that enqueues many short launches per step (CG's
// batches) is captured once and replayed, so the host pays one launch per
// batch instead of several per iteration.
struct svb_graph {
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;   // kernel nodes, counted into svb_launch_count per replay
};
int svb_graph_begin(void* stream) {
  return guard([&] { SVB_CUDA_TRY(cudaStreamBeginCapture(S(stream), cudaStreamCaptureModeThreadLocal)); });
}
int svb_graph_end(void* stream, void** out) {
  return guard([&] {
    cudaGraph_t g = nullptr;
    SVB_CUDA_TRY(cudaStreamEndCapture(S(stream), &g));
    auto* h = new svb_graph();
    size_t nn = 0;
    SVB_CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) SVB_CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      SVB_CUDA_TRY(cudaGraphNodeGetType(nd, &t));
      h->kernels += t == cudaGraphNodeTypeKernel;
    }
    const cudaError_t e = cudaGraphInstantiate(&h->exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      delete h;
      SVB_CUDA_TRY(e);
    }
    // the captured launches were counted once at capture time; replays count again
    note_launches(-h->kernels);
    *out = h;
  });
}
int svb_graph_launch(void* graph, void* stream) {
  return guard([&] {
    auto* h = static_cast<svb_graph*>(graph);
    SVB_CUDA_TRY(cudaGraphLaunch(h->exec, S(stream)));
    note_launches(h->kernels);
  });
}
int svb_graph_destroy(void* graph) {
  return guard([&] {
    auto* h = static_cast<svb_graph*>(graph);
    if (h && h->exec) cudaGraphExecDestroy(h->exec);
    delete h;
  });
}

int svb_event_record(void* stream, void** out) {
  return guard([&] {
    cudaEvent_t e;
    SVB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SVB_CUDA_TRY(cudaEventRecord(e, S(stream)));
    *out = e;
  });
}
int svb_event_sync(void* event) {
  return guard([&] { SVB_CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(event))); });
}
int svb_event_query(void* event) {
  cudaError_t e = cudaEventQuery(reinterpret_cast<cudaEvent_t>(event));
  if (e == cudaSuccess) return SVB_OK;
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    return SVB_INVALID;
  }
  set_error(cudaGetErrorString(e));
  return SVB_CUDA;
}
int svb_stream_wait_event(void* stream, void* event) {
  return guard([&] { SVB_CUDA_TRY(cudaStreamWaitEvent(S(stream), reinterpret_cast<cudaEvent_t>(event), 0)); });
}
int svb_event_destroy(void* event) {
  return guard([&] { SVB_CUDA_TRY(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event))); });
}
int svb_malloc(int64_t bytes, void** out) {
  return guard([&] {
    *out = nullptr;
    if (bytes > 0) SVB_CUDA_TRY(cudaMallocAsync(out, bytes, 0));
    SVB_CUDA_TRY(cudaStreamSynchronize(0));
  });
}
int svb_free(void* p) {
  return guard([&] {
    if (!p) return;
    SVB_CUDA_TRY(cudaDeviceSynchronize());
    SVB_CUDA_TRY(cudaFreeAsync(p, 0));
  });
}
int svb_host_alloc(int64_t bytes, void** out) {
  return guard([&] { SVB_CUDA_TRY(cudaHostAlloc(out, bytes > 0 ? bytes : 1, cudaHostAllocDefault)); });
}
int svb_host_free(void* p) {
  return guard([&] { SVB_CUDA_TRY(cudaFreeHost(p)); });
}
int svb_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  return guard([&] {
    if (bytes > 0) SVB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, S(stream)));
  });
}
int svb_copy_host(void* dst, const void* src, int64_t bytes, int32_t to_device, void* stream) {
  return guard([&] {
    if (bytes <= 0) return;
    cudaStream_t s = S(stream);
    const void* host = to_device ? src : dst;
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();   // an unregistered pointer is not an error here
    if (pinned || to_device || bytes < STAGE_MIN) {
      SVB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
      return;
    }
    int dev = 0;
    SVB_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(g_stage_mu);
    char* ring = stage_buffer(std::min(bytes, STAGE_MAX));
    const int T = stage_threads();
    char* d = static_cast<char*>(dst);
    const char* h = static_cast<const char*>(src);
    for (int64_t off = 0; off < bytes; off += STAGE_MAX) {
      const int64_t win = std::min(STAGE_MAX, bytes - off);
      const int64_t part = (((win + T - 1) / T) + 4095) & ~int64_t(4095);
      std::vector<cudaEvent_t> ev(T, nullptr);
      std::atomic<int> err{0};
      if (!to_device) {   // all parts' DMAs first, in order; each thread drains one
        for (int t = 0; t < T && t * part < win; ++t) {
          const int64_t lo = t * part, len = std::min(part, win - lo);
          SVB_CUDA_TRY(cudaMemcpyAsync(ring + lo, h + off + lo, len, cudaMemcpyDeviceToHost, s));
          SVB_CUDA_TRY(cudaEventCreateWithFlags(&ev[t], cudaEventDisableTiming));
          SVB_CUDA_TRY(cudaEventRecord(ev[t], s));
        }
      }
      std::vector<std::thread> th;
      for (int t = 0; t < T && t * part < win; ++t) {
        th.emplace_back([&, t] {
          const int64_t lo = t * part, len = std::min(part, win - lo);
          if (cudaSetDevice(dev) != cudaSuccess) {
            err = 1;
            return;
          }
          if (to_device) {
            std::memcpy(ring + lo, h + off + lo, len);
            if (cudaMemcpyAsync(d + off + lo, ring + lo, len, cudaMemcpyHostToDevice, s) != cudaSuccess) err = 1;
          } else {
            if (cudaEventSynchronize(ev[t]) != cudaSuccess) {
              err = 1;
              return;
            }
            std::memcpy(d + off + lo, ring + lo, len);
          }
        });
      }
      for (auto& x : th) x.join();
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
      if (to_device) SVB_CUDA_TRY(cudaStreamSynchronize(s));   // the staging buffer is free again
      SVB_REQUIRE(err.load() == 0, SVB_CUDA, "staged host copy failed");
    }
  });
}
int svb_memset(void* dst, int value, int64_t bytes, void* stream) {
  return guard([&] {
    if (bytes > 0) SVB_CUDA_TRY(cudaMemsetAsync(dst, value, bytes, S(stream)));
  });
}
int svb_pool_info(int64_t* reserved, int64_t* used) {
  return guard([&] {
    int dev = 0;
    SVB_CUDA_TRY(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    SVB_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t r = 0, u = 0;
    SVB_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r));
    SVB_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
    *reserved = (int64_t)r;
    *used = (int64_t)u;
  });
}

int svb_device_info(int32_t* sms, int64_t* free_b, int64_t* total_b) {
  return guard([&] {
    size_t f = 0, t = 0;
    SVB_CUDA_TRY(cudaMemGetInfo(&f, &t));
    *sms = sm_count();
    *free_b = (int64_t)f;
    *total_b = (int64_t)t;
  });
}

int svb_coo_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows_host,
                   const int64_t* cols_host, const double* vals_host, void* stream,
                   svb_matrix** out) {
  return guard([&] {
    require_index_range(nrows, ncols);
    cudaStream_t s = S(stream);
    auto m = new svb_matrix();
    m->fmt = SVB_COO;
    m->nrows = nrows; m->ncols = ncols; m->nnz = nnz;
    m->ptr64 = want_ptr64(nnz);
    m->rows = upload_i32(rows_host, nnz, s);
    m->cols = upload_i32(cols_host, nnz, s);
    m->vals = upload(vals_host, nnz * 8, s);
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(m);
  });
}

int svb_csr_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row_ptr_host,
                   const int64_t* col_idx_host, const double* vals_host, void* stream,
                   svb_matrix** out) {
  return guard([&] {
    require_index_range(nrows, ncols);
    cudaStream_t s = S(stream);
    auto m = new svb_matrix();
    m->fmt = SVB_CSR;
    m->nrows = nrows; m->ncols = ncols; m->nnz = nnz;
    m->ptr64 = want_ptr64(nnz);
    if (m->ptr64) m->ptr = upload(row_ptr_host, (nrows + 1) * 8, s);
    else m->ptr = upload_i32(row_ptr_host, nrows + 1, s);
    m->cols = upload_i32(col_idx_host, nnz, s);
    m->vals = upload(vals_host, nnz * 8, s);
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(m);
  });
}

int svb_csr_create_slab(int64_t nrows, int64_t ncols_global, int64_t nnz, int64_t r0, const int64_t* row_ptr_host,
                        const void* col_idx_host, int32_t cols_i64, const double* vals_host, void* stream,
                        int64_t* window, svb_matrix** out) {
  return guard([&] {
    require_index_range(nrows, ncols_global);
    SVB_REQUIRE(r0 >= 0 && r0 + nrows <= ncols_global, SVB_DIM_MISMATCH, "slab rows outside the matrix");
    SVB_REQUIRE(nnz >= 0 && window && out, SVB_INVALID, "slab: null output or negative nnz");
    SVB_REQUIRE(row_ptr_host[0] == 0 && row_ptr_host[nrows] == nnz, SVB_DIM_MISMATCH,
                "row_ptr endpoints must be 0 and nnz");
    cudaStream_t s = S(stream);
    std::unique_ptr<svb_matrix> m(new svb_matrix());
    m->fmt = SVB_CSR;
    m->nrows = nrows;
    m->nnz = nnz;
    m->ptr64 = want_ptr64(nnz);
    m->ptr = m->ptr64 ? upload(row_ptr_host, (nrows + 1) * 8, s) : upload_i32(row_ptr_host, nrows + 1, s);
    // columns: the global indices land in a staging buffer (int64) or in
    // place (int32); their hull with the own rows is the rank's window
    Buf stage;
    if (cols_i64) stage = upload(col_idx_host, nnz * 8, s);
    m->cols = cols_i64 ? alloc(nnz * 4, s) : upload(col_idx_host, nnz * 4, s);
    Buf mm = alloc(16 + 8, s);
    long long init[2] = {LLONG_MAX, LLONG_MIN};
    SVB_CUDA_TRY(cudaMemcpyAsync(mm->ptr, init, 16, cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
      if (cols_i64)
        k_col_minmax<int64_t><<<grid_for(nnz, 256, 4), 256, 0, s>>>(ptr<int64_t>(stage), nnz, ptr<long long>(mm));
      else
        k_col_minmax<int32_t><<<grid_for(nnz, 256, 4), 256, 0, s>>>(ptr<int32_t>(m->cols), nnz, ptr<long long>(mm));
      SVB_CHECK_LAUNCH();
    }
    long long got[2];
    SVB_CUDA_TRY(cudaMemcpyAsync(got, mm->ptr, 16, cudaMemcpyDeviceToHost, s));
    m->vals = upload(vals_host, nnz * 8, s);   // the H2D of values overlaps nothing else; keep it queued
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    if (nnz > 0)
      SVB_REQUIRE(got[0] >= 0 && got[1] < ncols_global, SVB_DIM_MISMATCH, "column index out of range");
    const int64_t cmin = nnz > 0 ? std::min<int64_t>(got[0], r0) : r0;
    const int64_t cmax = nnz > 0 ? std::max<int64_t>(got[1], r0 + nrows - 1) : r0 + nrows - 1;
    SVB_REQUIRE(cmax - cmin + 1 < INT32_MAX, SVB_INAPPLICABLE,
                "slab column window >= 2^31 is not supported by the int32 device index layout");
    if (nnz > 0 && (cols_i64 || cmin != 0)) {
      if (cols_i64)
        k_cols_rebase<int64_t><<<grid_for(nnz, 256), 256, 0, s>>>(ptr<int64_t>(stage), ptr<int32_t>(m->cols), nnz, cmin);
      else
        k_cols_rebase<int32_t><<<grid_for(nnz, 256), 256, 0, s>>>(ptr<int32_t>(m->cols), ptr<int32_t>(m->cols), nnz, cmin);
      SVB_CHECK_LAUNCH();
    }
    stage.reset();
    m->ncols = cmax - cmin + 1;
    int* flags = reinterpret_cast<int*>(mm->ptr);
    SVB_CUDA_TRY(cudaMemsetAsync(flags, 0, 8, s));
    if (m->ptr64)
      k_csr_check<int64_t><<<grid_for(nrows, 256), 256, 0, s>>>(nrows, ptr<int64_t>(m->ptr), ptr<int32_t>(m->cols), flags);
    else
      k_csr_check<int32_t><<<grid_for(nrows, 256), 256, 0, s>>>(nrows, ptr<int32_t>(m->ptr), ptr<int32_t>(m->cols), flags);
    SVB_CHECK_LAUNCH();
    int fl[2];
    SVB_CUDA_TRY(cudaMemcpyAsync(fl, flags, 8, cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    SVB_REQUIRE(!fl[0], SVB_DIM_MISMATCH, "row_ptr must be non-decreasing");
    SVB_REQUIRE(!fl[1], SVB_DIM_MISMATCH, "columns not strictly increasing within a row");
    window[0] = cmin;
    window[1] = cmax;
    *out = publish(m.release());
  });
}

int svb_csr_export(const svb_matrix* m, int64_t col_shift, int64_t* row_ptr_host, int32_t* cols_host,
                   double* vals_host, void* stream) {
  return guard([&] {
    SVB_REQUIRE(m && m->fmt == SVB_CSR, SVB_UNSUPPORTED_CONFIG, "export needs a CSR matrix");
    cudaStream_t s = S(stream);
    {
      Buf p64 = alloc((m->nrows + 1) * 8, s);
      ptr_to_i64(m, ptr<int64_t>(p64), s);
      SVB_CUDA_TRY(cudaMemcpyAsync(row_ptr_host, p64->ptr, (m->nrows + 1) * 8, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
    }
    // chunked: shift a piece of the columns on the device, copy it down
    constexpr int64_t CH = int64_t(1) << 27;   // 128 Mi entries (512 MB)
    Buf tmp = col_shift ? alloc(std::min(m->nnz, CH) * 4 + 4, s) : Buf();
    for (int64_t o = 0; o < m->nnz; o += CH) {
      const int64_t c = std::min(CH, m->nnz - o);
      const int32_t* src = ptr<int32_t>(m->cols) + o;
      if (col_shift) {
        k_cols_shift<<<grid_for(c, 256), 256, 0, s>>>(src, ptr<int32_t>(tmp), c, col_shift);
        SVB_CHECK_LAUNCH();
        src = ptr<int32_t>(tmp);
      }
      SVB_CUDA_TRY(cudaMemcpyAsync(cols_host + o, src, c * 4, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
    }
    if (m->nnz)
      SVB_CUDA_TRY(cudaMemcpyAsync(vals_host, m->vals->ptr, m->nnz * 8, cudaMemcpyDeviceToHost, s));
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
  });
}

int svb_csr_row_slice(const svb_matrix* src, int64_t r0, int64_t r1, void* stream,
                      svb_matrix** out) {
  return guard([&] {
    SVB_REQUIRE(src && src->fmt == SVB_CSR, SVB_UNSUPPORTED_CONFIG, "row slice needs a CSR matrix");
    SVB_REQUIRE(0 <= r0 && r0 < r1 && r1 <= src->nrows, SVB_DIM_MISMATCH,
                "row slice must be a non-empty range inside the matrix");
    cudaStream_t s = S(stream);
    int64_t b[2];
    if (src->ptr64) {
      SVB_CUDA_TRY(cudaMemcpyAsync(&b[0], ptr<int64_t>(src->ptr) + r0, 8, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaMemcpyAsync(&b[1], ptr<int64_t>(src->ptr) + r1, 8, cudaMemcpyDeviceToHost, s));
    } else {
      int32_t b32[2];
      SVB_CUDA_TRY(cudaMemcpyAsync(&b32[0], ptr<int32_t>(src->ptr) + r0, 4, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaMemcpyAsync(&b32[1], ptr<int32_t>(src->ptr) + r1, 4, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
      b[0] = b32[0]; b[1] = b32[1];
    }
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    auto m = new svb_matrix();
    m->fmt = SVB_CSR;
    m->nrows = r1 - r0; m->ncols = src->ncols; m->nnz = b[1] - b[0];
    m->ptr64 = want_ptr64(m->nnz);
    const int64_t n1 = m->nrows + 1;
    m->ptr = alloc(n1 * (m->ptr64 ? 8 : 4), s);
    const int g = grid_for(n1, 256);
    if (src->ptr64 && m->ptr64)
      k_rebase_ptr<<<g, 256, 0, s>>>(ptr<int64_t>(src->ptr) + r0, ptr<int64_t>(m->ptr), n1);
    else if (src->ptr64)
      k_rebase_ptr<<<g, 256, 0, s>>>(ptr<int64_t>(src->ptr) + r0, ptr<int32_t>(m->ptr), n1);
    else if (m->ptr64)   // SPMVTUNE_FORCE_PTR64 on an int32 source
      k_rebase_ptr<<<g, 256, 0, s>>>(ptr<int32_t>(src->ptr) + r0, ptr<int64_t>(m->ptr), n1);
    else
      k_rebase_ptr<<<g, 256, 0, s>>>(ptr<int32_t>(src->ptr) + r0, ptr<int32_t>(m->ptr), n1);
    SVB_CHECK_LAUNCH();
    m->cols = alloc(m->nnz * 4, s);
    m->vals = alloc(m->nnz * 8, s);
    if (m->nnz) {
      SVB_CUDA_TRY(cudaMemcpyAsync(m->cols->ptr, ptr<int32_t>(src->cols) + b[0], m->nnz * 4,
                                   cudaMemcpyDeviceToDevice, s));
      SVB_CUDA_TRY(cudaMemcpyAsync(m->vals->ptr, ptr<double>(src->vals) + b[0], m->nnz * 8,
                                   cudaMemcpyDeviceToDevice, s));
    }
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(m);
  });
}

int svb_ell_create(int64_t nrows, int64_t ncols, int64_t width, const int64_t* cols_host,
                   const double* vals_host, void* stream, svb_matrix** out) {
  return guard([&] {
    require_index_range(nrows, ncols);
    cudaStream_t s = S(stream);
    auto m = new svb_matrix();
    m->fmt = SVB_ELL;
    m->nrows = nrows; m->ncols = ncols; m->width = width;
    int64_t cells = nrows * width;
    m->cols = upload_i32(cols_host, cells, s);
    m->vals = upload(vals_host, cells * 8, s);
    int64_t stored = 0;
    for (int64_t i = 0; i < cells; ++i) stored += cols_host[i] != ncols;
    m->nnz = stored;
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(m);
  });
}

int svb_dia_create(int64_t nrows, int64_t ncols, int64_t ndiag, const int64_t* offsets_host,
                   const double* data_host, void* stream, svb_matrix** out) {
  return guard([&] {
    require_index_range(nrows, ncols);
    cudaStream_t s = S(stream);
    auto m = new svb_matrix();
    m->fmt = SVB_DIA;
    m->nrows = nrows; m->ncols = ncols; m->ndiag = ndiag;
    m->h_offs.assign(offsets_host, offsets_host + ndiag);
    m->offs = upload(offsets_host, ndiag * 8, s);
    m->vals = upload(data_host, ndiag * nrows * 8, s);
    int64_t stored = 0;  // in-range cells (DiaMatrix carries no nnz; informational)
    for (int64_t k = 0; k < ndiag; ++k) {
      int64_t off = offsets_host[k];
      int64_t lo = off < 0 ? -off : 0, hi = nrows < ncols - off ? nrows : ncols - off;
      if (hi > lo) stored += hi - lo;
    }
    m->nnz = stored;
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(m);
  });
}

int svb_hyb_create(const svb_matrix* ell, const svb_matrix* coo, void* stream, svb_matrix** out) {
  return guard([&] {
    SVB_REQUIRE(ell && coo && ell->fmt == SVB_ELL && coo->fmt == SVB_COO, SVB_INVALID,
                "HYB needs an ELL part and a COO part");
    SVB_REQUIRE(ell->nrows == coo->nrows && ell->ncols == coo->ncols, SVB_DIM_MISMATCH,
                "ELL and COO parts must share dimensions");
    cudaStream_t s = S(stream);
    auto m = new svb_matrix();
    m->fmt = SVB_HYB;
    m->nrows = ell->nrows; m->ncols = ell->ncols; m->width = ell->width;
    m->cols = ell->cols; m->vals = ell->vals;
    m->rows = coo->rows; m->scols = coo->cols; m->svals = coo->vals;
    m->spill_nnz = coo->nnz;
    m->nnz = ell->nnz + coo->nnz;
    m->ptr = rows_to_ptr(ptr<int32_t>(coo->rows), coo->nnz, coo->nrows, true, s);
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(m);
  });
}

int svb_matrix_destroy(svb_matrix* m) {
  // other streams may still read the buffers: drain the device first
  return guard([&] {
    SVB_CUDA_TRY(cudaDeviceSynchronize());
    forget_bounds(m);
    delete m;
  });
}

int svb_matrix_info_get(const svb_matrix* m, svb_matrix_info* info) {
  return guard([&] {
    SVB_REQUIRE(m && info, SVB_INVALID, "null handle");
    info->format = m->fmt;
    info->ptr64 = m->ptr64;
    info->nrows = m->nrows;
    info->ncols = m->ncols;
    info->nnz = m->nnz;
    info->width = m->width;
    info->ndiag = m->ndiag;
    info->spill_nnz = m->spill_nnz;
    info->device_bytes = m->device_bytes();
  });
}

int svb_matrix_download(const svb_matrix* m, int which, void* dst, void* stream) {
  return guard([&] {
    SVB_REQUIRE(m && dst, SVB_INVALID, "null handle");
    cudaStream_t s = S(stream);
    auto copy_i32 = [&](const Buf& b, int64_t n) {
      if (n <= 0) return;
      Buf w = alloc(n * 8, s);
      widen_i32_to_i64(ptr<int32_t>(b), ptr<int64_t>(w), n, s);
      SVB_CUDA_TRY(cudaMemcpyAsync(dst, w->ptr, n * 8, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
    };
    auto copy_raw = [&](const Buf& b, int64_t bytes) {
      if (bytes <= 0) return;
      SVB_CUDA_TRY(cudaMemcpyAsync(dst, b->ptr, bytes, cudaMemcpyDeviceToHost, s));
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
    };
    switch (which) {
      case SVB_ARR_ROW_PTR:
        SVB_REQUIRE(m->fmt == SVB_CSR || m->fmt == SVB_HYB, SVB_INVALID, "no row_ptr");
        if (m->fmt == SVB_HYB || m->ptr64) copy_raw(m->ptr, (m->nrows + 1) * 8);
        else copy_i32(m->ptr, m->nrows + 1);
        break;
      case SVB_ARR_ROWS:
        SVB_REQUIRE(m->fmt == SVB_COO || m->fmt == SVB_HYB, SVB_INVALID, "no rows array");
        copy_i32(m->rows, m->fmt == SVB_COO ? m->nnz : m->spill_nnz);
        break;
      case SVB_ARR_COLS:
        if (m->fmt == SVB_ELL || m->fmt == SVB_HYB) copy_i32(m->cols, m->width * m->nrows);
        else {
          SVB_REQUIRE(m->fmt == SVB_CSR || m->fmt == SVB_COO, SVB_INVALID, "no cols array");
          copy_i32(m->cols, m->nnz);
        }
        break;
      case SVB_ARR_VALS:
        if (m->fmt == SVB_ELL || m->fmt == SVB_HYB) copy_raw(m->vals, m->width * m->nrows * 8);
        else {
          SVB_REQUIRE(m->fmt == SVB_CSR || m->fmt == SVB_COO, SVB_INVALID, "no values array");
          copy_raw(m->vals, m->nnz * 8);
        }
        break;
      case SVB_ARR_OFFSETS:
        SVB_REQUIRE(m->fmt == SVB_DIA, SVB_INVALID, "no offsets");
        if (m->ndiag) std::memcpy(dst, m->h_offs.data(), m->ndiag * 8);
        break;
      case SVB_ARR_DATA:
        SVB_REQUIRE(m->fmt == SVB_DIA, SVB_INVALID, "no DIA data");
        copy_raw(m->vals, m->ndiag * m->nrows * 8);
        break;
      case SVB_ARR_SPILL_COLS:
        SVB_REQUIRE(m->fmt == SVB_HYB, SVB_INVALID, "no spill");
        copy_i32(m->scols, m->spill_nnz);
        break;
      case SVB_ARR_SPILL_VALS:
        SVB_REQUIRE(m->fmt == SVB_HYB, SVB_INVALID, "no spill");
        copy_raw(m->svals, m->spill_nnz * 8);
        break;
      default:
        throw Error{SVB_INVALID, "unknown array selector"};
    }
  });
}

}  // extern "C"
