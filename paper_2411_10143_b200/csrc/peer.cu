// Peer-memory collectives for the row-partitioned solvers (distributed.py):
// the per-iteration exchanges of the row-partitioned CG done by the solver's
// own kernels over NVLink / NVSwitch peer memory instead of NCCL calls.
//
//  * all-reduce of a few device scalars (CG's p.Ap and r.r, the CGS2 dot
//    blocks): every rank stores its values into slot [rank] of EVERY rank's
//    mailbox (remote stores over NVLink), fences at system scope and
//    release-stores a tag = the operation's epoch; each rank then spins on
//    the tags in its OWN mailbox (local reads) and sums the slots in rank
//    order, so every rank gets the bit-identical total.  Two slot banks by
//    epoch parity: a rank can only reach epoch e + 2 after every rank has
//    finished e + 1, hence after every rank has read bank e.
//  * halo push: the pass that produces the next search direction
//    (k_dcg_xp_push: x += a p, p = r + b p) stores the rows a neighbour
//    needs straight into the neighbour's window buffer, then its last CTA
//    release-stores a halo tag into the neighbour's mailbox; the
//    neighbour's boundary-row SpMV is preceded by k_peer_wait on that tag
//    (its interior rows run meanwhile).  The write-after-read hazard (my
//    push overwriting a halo my neighbour is still multiplying with) cannot
//    occur: the push follows the r.r all-reduce, which needs the
//    neighbour's contribution, which its stream enqueues after its SpMV.
//
// Every wait has a deadline (a mapped host error word is raised and the
// kernel returns), so a protocol fault surfaces as an error, never a hang.
// Buffers other ranks write into (mailboxes, windows) come from cudaMalloc
// so they can be exported with CUDA IPC; in one process they are plain
// device pointers.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace svb {

constexpr int PEER_MAXW = 8;    // ranks per group: one 8-GPU NVSwitch box
constexpr int PEER_MAXC = 64;   // doubles per all-reduce
constexpr unsigned long long PEER_DEADLINE_NS = 30ull * 1000000000ull;

struct Mailbox {
  unsigned long long ar_tag[2][PEER_MAXW];
  unsigned long long halo_tag[PEER_MAXW];
  double ar_val[2][PEER_MAXW][PEER_MAXC];
};

struct PeerView {
  int rank, world;
  Mailbox* mb[PEER_MAXW];   // every rank's mailbox as addressable from this GPU (own included)
  int* err;                 // mapped host word, raised by a wait that passed its deadline
  unsigned long long deadline_ns;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// spin until *p >= want; false (error word raised) past the deadline
__device__ bool spin_ge(const unsigned long long* p, unsigned long long want, int* err,
                        unsigned long long deadline_ns) {
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(p) < want) {
    if (*(volatile int*)err) return false;   // another wait already failed: stop too
    if (global_ns() - t0 > deadline_ns) {
      *(volatile int*)err = 1;
      __threadfence_system();
      return false;
    }
    __nanosleep(100);
  }
  return true;
}

// v[0..count) <- sum over ranks (rank order), one CTA
__global__ void k_peer_allreduce(double* v, int count, PeerView pv, unsigned long long epoch) {
  const int par = (int)(epoch & 1), tid = threadIdx.x, me = pv.rank;
  for (int q = 0; q < pv.world; ++q)
    for (int c = tid; c < count; c += blockDim.x) pv.mb[q]->ar_val[par][me][c] = v[c];
  __threadfence_system();
  __syncthreads();
  if (tid < pv.world) st_release_sys(&pv.mb[tid]->ar_tag[par][me], epoch);
  if (tid < pv.world) spin_ge(&pv.mb[me]->ar_tag[par][tid], epoch, pv.err, pv.deadline_ns);
  __syncthreads();
  __threadfence_system();
  const Mailbox* own = pv.mb[me];
  for (int c = tid; c < count; c += blockDim.x) {
    double s = ld_relaxed_sys(&own->ar_val[par][0][c]);
    for (int q = 1; q < pv.world; ++q) s += ld_relaxed_sys(&own->ar_val[par][q][c]);
    v[c] = s;
  }
}

// wait until every listed peer has pushed halo `epoch` into this rank's window
__global__ void k_peer_wait(PeerView pv, int npeers, int p0, int p1, unsigned long long epoch) {
  const int t = threadIdx.x;
  if (t < npeers) spin_ge(&pv.mb[pv.rank]->halo_tag[t == 0 ? p0 : p1], epoch, pv.err, pv.deadline_ns);
  __syncthreads();
}

struct PushSeg {
  int64_t lo, cnt;   // local rows [lo, lo + cnt) of this rank ...
  double* dst;       // ... stored to dst[0 .. cnt) in the peer's window
  int peer;
};
struct PushArgs {
  int nseg;
  PushSeg seg[2];
  unsigned long long epoch;
  unsigned* counter;   // zero between launches
};

// x += a p, then p = r + b p (a = sc[ialpha], b = sc[inew]/sc[iold]; the
// k_dcg_xp arithmetic), the new p of the rows a neighbour reads also stored
// into its window; the last CTA to finish signals the neighbours.
__global__ void __launch_bounds__(256) k_dcg_xp_push(int64_t n, const double* sc, int ialpha, int inew, int iold,
                                                     const double* __restrict__ r, double* __restrict__ p,
                                                     double* __restrict__ x, PushArgs pa, PeerView pv) {
  const double a = sc[ialpha];
  const double b = sc[inew] / sc[iold];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double pe = p[e];
    x[e] = x[e] + a * pe;
    const double pn = r[e] + b * pe;
    p[e] = pn;
#pragma unroll
    for (int s = 0; s < 2; ++s)
      if (s < pa.nseg && (uint64_t)(e - pa.seg[s].lo) < (uint64_t)pa.seg[s].cnt) pa.seg[s].dst[e - pa.seg[s].lo] = pn;
  }
  __threadfence_system();   // this thread's remote stores before the CTA's arrival
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(pa.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int s = 0; s < pa.nseg; ++s) st_release_sys(&pv.mb[pa.seg[s].peer]->halo_tag[pv.rank], pa.epoch);
    *pa.counter = 0;
  }
}

}  // namespace svb

using namespace svb;

struct svb_peer {
  PeerView view{};
  Mailbox* own = nullptr;                 // this rank's mailbox (cudaMalloc)
  int* err_host = nullptr;                // mapped error word
  unsigned* counter = nullptr;            // k_dcg_xp_push arrival counter
  unsigned long long ar_epoch = 0, halo_epoch = 0;
};

extern "C" {

int svb_peer_create(int rank, int world, svb_peer** out) {
  return guard([&] {
    SVB_REQUIRE(out && world >= 1 && world <= PEER_MAXW && rank >= 0 && rank < world, SVB_INVALID,
                "peer group: 1 <= world <= 8 and 0 <= rank < world");
    auto* g = new svb_peer();
    try {
      SVB_CUDA_TRY(cudaMalloc((void**)&g->own, sizeof(Mailbox)));
      SVB_CUDA_TRY(cudaMemset(g->own, 0, sizeof(Mailbox)));
      SVB_CUDA_TRY(cudaMalloc((void**)&g->counter, 16));
      SVB_CUDA_TRY(cudaMemset(g->counter, 0, 16));
      SVB_CUDA_TRY(cudaHostAlloc((void**)&g->err_host, sizeof(int), cudaHostAllocMapped));
      *g->err_host = 0;
      int* err_dev = nullptr;
      SVB_CUDA_TRY(cudaHostGetDevicePointer((void**)&err_dev, g->err_host, 0));
      SVB_CUDA_TRY(cudaDeviceSynchronize());
      g->view.rank = rank;
      g->view.world = world;
      g->view.err = err_dev;
      // SPMVTUNE_PEER_DEADLINE_MS shortens the wait deadline (tests of the error path)
      const char* dl = std::getenv("SPMVTUNE_PEER_DEADLINE_MS");
      g->view.deadline_ns = dl ? (unsigned long long)std::atoll(dl) * 1000000ull : PEER_DEADLINE_NS;
      g->view.mb[rank] = g->own;
    } catch (...) {
      if (g->own) cudaFree(g->own);
      if (g->counter) cudaFree(g->counter);
      if (g->err_host) cudaFreeHost(g->err_host);
      delete g;
      throw;
    }
    *out = g;
  });
}

int svb_peer_destroy(svb_peer* g) {
  return guard([&] {
    if (!g) return;
    cudaDeviceSynchronize();
    cudaFree(g->own);
    cudaFree(g->counter);
    cudaFreeHost(g->err_host);
    delete g;
  });
}

int svb_peer_mailbox(const svb_peer* g, void** dev_ptr) {
  return guard([&] {
    SVB_REQUIRE(g && dev_ptr, SVB_INVALID, "null argument");
    *dev_ptr = g->own;
  });
}

// rank q's mailbox as addressable here: a device pointer (same process) or
// an IPC handle opened with svb_peer_ipc_open
int svb_peer_set_mailbox(svb_peer* g, int q, void* dev_ptr) {
  return guard([&] {
    SVB_REQUIRE(g && dev_ptr && q >= 0 && q < g->view.world, SVB_INVALID, "bad peer mailbox");
    g->view.mb[q] = static_cast<Mailbox*>(dev_ptr);
  });
}

int svb_peer_alloc(int64_t bytes, void** out) {
  return guard([&] {
    SVB_REQUIRE(out && bytes >= 0, SVB_INVALID, "bad allocation request");
    SVB_CUDA_TRY(cudaMalloc(out, (size_t)std::max<int64_t>(bytes, 16) + 128));
    SVB_CUDA_TRY(cudaMemset(*out, 0, (size_t)std::max<int64_t>(bytes, 16) + 128));
  });
}

int svb_peer_free(void* p) {
  return guard([&] {
    if (p) {
      SVB_CUDA_TRY(cudaDeviceSynchronize());
      SVB_CUDA_TRY(cudaFree(p));
    }
  });
}

// 64-byte CUDA IPC handle of a cudaMalloc'd pointer (svb_peer_alloc, a mailbox)
int svb_peer_ipc_handle(void* dev_ptr, void* handle64) {
  return guard([&] {
    SVB_REQUIRE(dev_ptr && handle64, SVB_INVALID, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    SVB_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
    std::memcpy(handle64, &h, 64);
  });
}

int svb_peer_ipc_open(const void* handle64, void** dev_ptr) {
  return guard([&] {
    SVB_REQUIRE(handle64 && dev_ptr, SVB_INVALID, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    SVB_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int svb_peer_ipc_close(void* dev_ptr) {
  return guard([&] {
    if (dev_ptr) SVB_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  });
}

int svb_peer_error(const svb_peer* g, int* err) {
  return guard([&] {
    SVB_REQUIRE(g && err, SVB_INVALID, "null argument");
    *err = *(volatile int*)g->err_host;
  });
}

// in-place sum over ranks of v_dev[0..count), enqueued on `stream`
int svb_peer_allreduce(svb_peer* g, double* v_dev, int count, void* stream) {
  return guard([&] {
    SVB_REQUIRE(g && v_dev && count >= 1 && count <= PEER_MAXC, SVB_INVALID, "peer all-reduce: 1..64 doubles");
    for (int q = 0; q < g->view.world; ++q) SVB_REQUIRE(g->view.mb[q], SVB_INVALID, "peer mailbox not set");
    const unsigned long long e = ++g->ar_epoch;
    k_peer_allreduce<<<1, 64, 0, reinterpret_cast<cudaStream_t>(stream)>>>(v_dev, count, g->view, e);
    SVB_CHECK_LAUNCH();
  });
}

// the stream waits (device side) for the halo the listed peers pushed with
// their latest svb_dcg_xp_push
int svb_peer_wait_halo(svb_peer* g, const int32_t* peers, int npeers, void* stream) {
  return guard([&] {
    SVB_REQUIRE(g && npeers >= 0 && npeers <= 2 && (npeers == 0 || peers), SVB_INVALID, "peer wait: <= 2 peers");
    if (npeers == 0) return;
    k_peer_wait<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(g->view, npeers, peers[0],
                                                                       npeers > 1 ? peers[1] : 0, g->halo_epoch);
    SVB_CHECK_LAUNCH();
  });
}

// x += sc[ialpha] p, p = r + (sc[inew]/sc[iold]) p over n local rows; rows
// [lo[s], lo[s] + cnt[s]) also stored to dst[s] (peer peer[s]'s window)
int svb_dcg_xp_push(svb_peer* g, int64_t n, const double* sc, int32_t ialpha, int32_t inew, int32_t iold,
                    const double* r, double* p, double* x, int nseg, const int64_t* lo, const int64_t* cnt,
                    double* const* dst, const int32_t* peer, void* stream) {
  return guard([&] {
    SVB_REQUIRE(g && nseg >= 0 && nseg <= 2, SVB_INVALID, "x/p push: at most 2 halo segments");
    PushArgs pa{};
    pa.nseg = nseg;
    for (int s = 0; s < nseg; ++s) {
      SVB_REQUIRE(lo[s] >= 0 && cnt[s] >= 0 && lo[s] + cnt[s] <= n && dst[s], SVB_INVALID, "bad halo segment");
      SVB_REQUIRE(peer[s] >= 0 && peer[s] < g->view.world && g->view.mb[peer[s]], SVB_INVALID, "bad halo peer");
      pa.seg[s] = PushSeg{lo[s], cnt[s], dst[s], peer[s]};
    }
    pa.epoch = ++g->halo_epoch;
    pa.counter = g->counter;
    const unsigned grid = grid_for(std::max<int64_t>(n, 1), 256, 8);
    k_dcg_xp_push<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n, sc, ialpha, inew, iold, r, p, x, pa,
                                                                           g->view);
    SVB_CHECK_LAUNCH();
  });
}

}  // extern "C"
