// TMA-streamed, TMEM-resident modified Gram-Schmidt for one Arnoldi step
// (reference _gmres_core, solver.py:294-313: for i <= j: h_i = V_i . w;
// w -= h_i V_i; then hnext = ||w||, V[j+1] = w / hnext).
//
// Persistent cooperative kernel, one CTA per SM; CTA c owns the slice
// [c*chunk, c*chunk + len) of every vector.
//
//  * w lives in tensor memory for the whole step (128 lanes x 512 columns =
//    32K doubles per SM); it never round-trips through L2/HBM.
//  * One producer thread streams the step's vectors through a ring of
//    shared-memory stages with 1-D bulk copies (TMA engine) completed on
//    mbarriers.  Pass i's stage pairs a chunk of V_{i-1} (second use, an L2
//    hit: it was streamed in by pass i-1) with the same chunk of V_i (HBM).
//    The producer runs ahead across pass boundaries, so while the consumers
//    sit in a grid barrier the ring keeps filling with the next pass's rows:
//    the HBM stream does not stop for the barrier.
//  * 16 consumer warps apply w -= h_{i-1} V_{i-1} and accumulate V_i . w
//    chunk by chunk, reading w from / writing it back to TMEM.
//  * The grid reduction is a tag exchange: each CTA publishes its partial
//    in self-validating tagged words and polls every CTA's slot; all CTAs
//    fold the partials in the same fixed order, so every CTA holds the
//    bit-identical h_i without a broadcast, atomics or memory fences.  Tags
//    carry a per-launch epoch, so no reset is needed between launches.
//
// HBM traffic per step: w once, each V_i once, V[j+1] written once:
// 8n(j+3) bytes, the algorithmic minimum.
//
// Slices longer than the on-chip capacity (MAXCH chunks: n > 148 x 32768 =
// 4.85 M rows) run partially resident: chunks [0, nres) as above, chunks
// [nres, nch) ("overflow") keep w in global memory — in the V[j+1] row it
// will be normalised into, each consumer thread loading and storing only its
// own elements (program order makes its stores visible to its next loads) —
// and re-stream V_{i-1} next to V_i instead of parking it in TMEM: 32 bytes
// per overflow element per pass instead of 8, against the 32n of the
// streaming fallback for every element.
#pragma once

#include <cstdint>

#include "spmvtune_b200.h"

namespace svb {
namespace mgs {

constexpr int CW = 8;                   // consumer warps (2 column blocks x 4 TMEM lane quadrants)
constexpr int U = 8;                    // doubles per consumer thread per chunk
constexpr int GQ = 2;                   // chunks per TMEM load/store group (x32 = 16 doubles)
constexpr int CT = CW * 32;             // consumer threads
constexpr int NT = CT + 32;             // + one producer warp (the HBM stream)
constexpr int E = 2048;                 // elements per chunk / ring stage (16 KB)
constexpr int MAXCH = 16;               // chunks per slice the TMEM layout can hold
constexpr int R = 6;                    // chunks of w held in registers (U doubles each per thread)
constexpr int R_OV = 4;                 // ... in the overflow mode (its prefetch registers)
constexpr int MAXCH_RES_OV = 14;        // chunks kept on chip in the overflow mode (same shared memory)
constexpr int NSB_MAX = 12;             // ring stages at most
constexpr int64_t MAX_SLICE = (int64_t)E * MAXCH;   // 32768 doubles = 256 KB of TMEM
constexpr int TCOLS = 512;
constexpr int SLOT_STRIDE = 32;         // words between exchange slots (256 B)
constexpr int HDR = 1024;               // barriers + scratch + TMEM base, ahead of w / ring
constexpr size_t SMEM = 232448;         // the whole opt-in shared memory: one CTA per SM
constexpr int MAXCH_OV = 64;            // chunks per slice with overflow (n <= 148 x 131072 = 19.4 M)

struct Args {
  double* V;            // basis rows, row stride ld
  int64_t n, ld, chunk;
  int m, j;
  double* H;            // (m+1) x m, column j written
  double* cs;
  double* sn;
  double* g;
  svb_krylov_status* st;   // mapped status block
  double bnorm;
  unsigned long long* gslot;  // [2][grid][SLOT_STRIDE] tagged partials (grid_exchange)
  unsigned long long epoch;   // distinct per launch
  int chunk_count;             // chunks in a full slice (plan())
  int nsb;                     // ring stages (plan())
  int nres;                    // chunks of a slice kept on chip (plan(); < chunk_count: overflow mode)
  unsigned long long* trace;  // optional: [grid][npass][4] globaltimer stamps (profiling)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(s_u32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 4 doubles (8 columns) per thread, lanes of this warp's quadrant
__device__ __forceinline__ void t_ld(uint32_t a, double (&v)[4]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a)
               : "memory");
}
// wait for this thread's outstanding tcgen05.ld; `v` is tied in as a
// read-write operand so no read of the loaded registers can be scheduled
// above the wait
__device__ __forceinline__ void t_wait_ld(double (&v)[4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+d"(v[0]), "+d"(v[1]), "+d"(v[2]), "+d"(v[3])::"memory");
}
__device__ __forceinline__ void t_st(uint32_t a, const double (&v)[4]) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(a), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// 16 doubles (32 columns) per thread: chunks 4g..4g+3 of this warp
__device__ __forceinline__ void t_ld32(uint32_t a, double (&v)[16]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(a)
      : "memory");
}
__device__ __forceinline__ void t_wait_ld16(double (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+d"(v[0]), "+d"(v[1]), "+d"(v[2]), "+d"(v[3]), "+d"(v[4]), "+d"(v[5]), "+d"(v[6]), "+d"(v[7]),
                 "+d"(v[8]), "+d"(v[9]), "+d"(v[10]), "+d"(v[11]), "+d"(v[12]), "+d"(v[13]), "+d"(v[14]), "+d"(v[15])
               :
               : "memory");
}
__device__ __forceinline__ void t_st32(uint32_t a, const double (&v)[16]) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(a),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void t_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Givens update of column j and the residual estimate (solver.py:300-313)
__device__ __forceinline__ void givens(const Args& A, double hnext) {
  const int m = A.m, j = A.j;
  double* H = A.H;
  for (int i = 0; i < j; ++i) {
    const double a = H[i * m + j], b = H[(i + 1) * m + j];
    const double hi = A.cs[i] * a + A.sn[i] * b;
    H[(i + 1) * m + j] = -A.sn[i] * a + A.cs[i] * b;
    H[i * m + j] = hi;
  }
  const double hjj = H[j * m + j];
  const double denom = hypot(hjj, hnext);
  double c = 1.0, s = 0.0;
  if (denom != 0.0) {
    c = hjj / denom;
    s = hnext / denom;
  }
  A.cs[j] = c;
  A.sn[j] = s;
  H[j * m + j] = c * hjj + s * hnext;
  A.g[j + 1] = -s * A.g[j];
  A.g[j] = c * A.g[j];
  H[(j + 1) * m + j] = hnext;
  const double est = fabs(A.g[j + 1]) / A.bnorm;
  A.st->hnext = hnext;
  A.st->hjj = H[j * m + j];
  A.st->estimate = est;
  A.st->nonfinite = !isfinite(hnext) || !isfinite(est);
}

// Grid-wide fixed-order sum of one value per CTA (consumer warp 0 only).
// Each CTA publishes its partial as two 64-bit words {tag:32 | half:32}
// (high and low halves of the double).  A 64-bit store is single-copy
// atomic, so a reader that sees the expected tag in both words holds the
// matching payload: no fences, no atomics, one L2 round trip to publish and
// one per poll.  The tag is (epoch:24 | pass+1:8); a slot is only ever
// overwritten by a later pass of the same launch or by the next launches,
// so a stale tag can never match.
__device__ __forceinline__ double grid_exchange(const Args& A, double part, int pass) {
  const int lane = threadIdx.x & 31;
  const unsigned G = gridDim.x;
  unsigned long long* slots = A.gslot + (size_t)(pass & 1) * SLOT_STRIDE * G;
  const unsigned long long want = ((A.epoch << 8) | (unsigned long long)(pass + 1)) & 0xffffffffull;
  if (lane == 0) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(part);
    const unsigned long long w0 = (want << 32) | (bits >> 32), w1 = (want << 32) | (bits & 0xffffffffull);
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slots + SLOT_STRIDE * blockIdx.x), "l"(w0),
                 "l"(w1)
                 : "memory");
  }
  // Slots are SLOT_STRIDE words apart so they hash to different L2 slices,
  // and a lane stops re-reading a slot once it holds the expected tag: the
  // poll traffic does not pile onto the slices the last publishers write.
  double v[8];
  unsigned pending = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[k] = 0.0;
    if (lane + 32 * k < G) pending |= 1u << k;
  }
  while (__any_sync(0xffffffffu, pending != 0)) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (pending & (1u << k)) {
        unsigned long long w0, w1;
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                     : "=l"(w0), "=l"(w1)
                     : "l"(slots + SLOT_STRIDE * (lane + 32 * k))
                     : "memory");
        if ((w0 >> 32) == want && (w1 >> 32) == want) {
          v[k] = __longlong_as_double((long long)((w0 << 32) | (w1 & 0xffffffffull)));
          pending &= ~(1u << k);
        }
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  return wsum(s);
}

// Consumer element layout: within a chunk, consumer thread c (0..CT-1)
// owns the element pairs 2c + 2*CT*i (+0, +1), i < U/2, so every shared
// memory access is a conflict-free 16-byte access (a warp covers 512
// contiguous bytes).  In TMEM the thread keeps its values in its own lane
// (32*(warp%4) + lane) at columns 256*(warp/4) + 16*q + 4i (+0..3).
struct Pair {
  double x, y;
};

__device__ __forceinline__ Pair lds2(const double* p) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}
__device__ __forceinline__ void sts2(double* p, double x, double y) {
  *reinterpret_cast<double2*>(p) = make_double2(x, y);
}

// OV: the partially resident (overflow) mode; OV = false compiles the
// fully resident kernel alone (no extra register pressure on its path)
template <bool OV>
__global__ void __launch_bounds__(NT, 1) k_mgs_tma(Args A) {
  constexpr int RR = OV ? R_OV : R;   // register-resident chunks of w
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);             // NSB_MAX
  uint64_t* empty = full + NSB_MAX;                                     // NSB_MAX
  double* scratch = reinterpret_cast<double*>(empty + NSB_MAX);        // 64 doubles
  uint32_t* tbase = reinterpret_cast<uint32_t*>(scratch + 64);
  double* wsm = reinterpret_cast<double*>(smem_raw + HDR);              // chunks RR.. of w

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t lo = (int64_t)blockIdx.x * A.chunk;
  const int64_t hi = A.n < lo + A.chunk ? A.n : lo + A.chunk;
  const int len = hi > lo ? (int)(hi - lo) : 0;
  const int nch = (len + E - 1) / E;
  const int nsb = A.nsb;
  const int nres = OV ? A.nres : A.chunk_count;
  const int nrc = OV ? (nch < nres ? nch : nres) : nch;   // this slice's resident chunks
  double* ring = wsm + (size_t)(nres > RR ? nres - RR : 0) * E;   // nsb x E
  const int j = A.j;
  const int npass = j + 2;   // pass 0 (w, V_0), passes 1..j (V_i), final

  if (threadIdx.x == 0) {
    for (int s = 0; s < nsb; ++s) {
      bar_init(full + s, 1);
      bar_init(empty + s, CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tbase)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  auto row = [&](int i) -> const double* { return A.V + (int64_t)i * A.ld + lo; };

  if (warp == CW) {
    // ---------------- producer: the step's HBM stream ----------------
    // pass 0: w chunk q, V_0 chunk q (interleaved); passes 1..j: V_p.
    // Nothing depends on h, so the ring refills while the consumers wait
    // in a grid exchange.
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      uint32_t ph = 0;
      auto put = [&](const double* src, int q) {
        bar_wait(empty + s, ph ^ 1);
        const int cnt = len - q * E < E ? len - q * E : E;
        const uint32_t bytes = (uint32_t)((cnt * 8 + 15) & ~15);
        bar_expect(full + s, bytes);
        g2s(ring + (size_t)s * E, src + (int64_t)q * E, bytes, full + s, pol);
        if (++s == nsb) {
          s = 0;
          ph ^= 1;
        }
      };
      for (int q = 0; q < nch; ++q) {
        if (!OV || q < nres) put(row(j + 1), q);   // overflow w is read by the consumers themselves
        put(row(0), q);
      }
      for (int p = 1; p <= j; ++p)
        for (int q = 0; q < nch; ++q) {
          if (OV && q >= nres) put(row(p - 1), q);   // V_{p-1} of overflow chunks: not in TMEM
          put(row(p), q);
        }
      if (OV)
        for (int q = nres; q < nch; ++q) put(row(j), q);   // final pass, overflow chunks
    }
    return;
  }

  // ---------------- consumers ----------------
  constexpr int NP = U / 2;   // pairs per thread per chunk
  const int qd = warp & 3, cg = warp >> 2;
  const uint32_t tw = *tbase + ((uint32_t)(32 * qd) << 16) + (uint32_t)(256 * cg);
  const int e0 = 2 * threadIdx.x;   // first element of pair 0 within a chunk
  double wr[RR][U];
  int rs = 0;
  uint32_t rph = 0;
  double h = 0.0;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  auto take = [&]() -> const double* {
    bar_wait(full + rs, rph);
    return ring + (size_t)rs * E + e0;
  };
  auto give = [&]() {
    __syncwarp();
    if (lane == 0) bar_arrive(empty + rs);
    if (++rs == nsb) {
      rs = 0;
      rph ^= 1;
    }
  };
  // element validity of pair i in a chunk with `lim` valid elements
  auto ok0 = [&](int i, int lim) { return e0 + 2 * CT * i < lim; };
  auto ok1 = [&](int i, int lim) { return e0 + 2 * CT * i + 1 < lim; };

  // One group of GQ chunks (g): TMEM load of V_{p-1} (32 columns), the
  // chunk updates, TMEM store of V_p.  W(k, i) is the address-or-register
  // accessor of this thread's w pair (chunk GQ*g+k, pair i).
#define MGS_GROUP(KIND, g, WLOAD, WSTORE)                                                           \
  {                                                                                             \
    double pv[GQ * U];                                                                          \
    const uint32_t ta = tw + (uint32_t)(32 * (g));                                              \
    if (KIND > 0) {                                                                             \
      t_ld32(ta, pv);                                                                           \
      t_wait_ld16(pv);                                                                          \
    }                                                                                           \
    _Pragma("unroll") for (int k = 0; k < GQ; ++k) {                                            \
      const int q = GQ * (g) + k;                                                               \
      if (q < nrc) {                                                                            \
        const int lim = len - q * E;                                                            \
        const bool fullc = lim >= E;                                                            \
        if (KIND == 0) {                                                                        \
          const double* sw = take();                                                            \
          double w[U];                                                                          \
          _Pragma("unroll") for (int i = 0; i < NP; ++i) {                                      \
            Pair t = lds2(sw + 2 * CT * i);                                                     \
            w[2 * i] = fullc || ok0(i, lim) ? t.x : 0.0;                                        \
            w[2 * i + 1] = fullc || ok1(i, lim) ? t.y : 0.0;                                    \
          }                                                                                     \
          give();                                                                               \
          const double* sv = take();                                                            \
          _Pragma("unroll") for (int i = 0; i < NP; ++i) {                                      \
            Pair t = lds2(sv + 2 * CT * i);                                                     \
            const double vx = fullc || ok0(i, lim) ? t.x : 0.0;                                 \
            const double vy = fullc || ok1(i, lim) ? t.y : 0.0;                                 \
            acc += vx * w[2 * i];                                                               \
            acc += vy * w[2 * i + 1];                                                           \
            pv[U * k + 2 * i] = vx;                                                             \
            pv[U * k + 2 * i + 1] = vy;                                                         \
            WSTORE(k, i, w[2 * i], w[2 * i + 1]);                                               \
          }                                                                                     \
          give();                                                                               \
        } else {                                                                                \
          const double* sv = KIND == 1 ? take() : nullptr;                                      \
          _Pragma("unroll") for (int i = 0; i < NP; ++i) {                                      \
            double wx, wy;                                                                      \
            WLOAD(k, i, wx, wy);                                                                \
            wx -= h * pv[U * k + 2 * i];                                                        \
            wy -= h * pv[U * k + 2 * i + 1];                                                    \
            if (KIND == 1) {                                                                    \
              Pair t = lds2(sv + 2 * CT * i);                                                   \
              const double vx = fullc || ok0(i, lim) ? t.x : 0.0;                               \
              const double vy = fullc || ok1(i, lim) ? t.y : 0.0;                               \
              acc += vx * wx;                                                                   \
              acc += vy * wy;                                                                   \
              pv[U * k + 2 * i] = vx;                                                           \
              pv[U * k + 2 * i + 1] = vy;                                                       \
            } else {                                                                            \
              acc += wx * wx;                                                                   \
              acc += wy * wy;                                                                   \
            }                                                                                   \
            WSTORE(k, i, wx, wy);                                                               \
          }                                                                                     \
          if (KIND == 1) give();                                                                \
        }                                                                                       \
      }                                                                                         \
    }                                                                                           \
    if (KIND < 2) t_st32(ta, pv);                                                               \
  }

  // overflow chunks [nres, nch): w in the V[j+1] row (this thread's own
  // pairs, loaded one chunk ahead), V_{p-1} streamed next to V_p
  double* wov = A.V + (int64_t)(j + 1) * A.ld + lo + e0;
  auto ov_load = [&](int q, double (&w)[U]) {
    const int lim = len - q * E;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const double* a = wov + (int64_t)q * E + 2 * CT * i;
      if (lim >= E || ok1(i, lim)) {
        const double2 t = __ldcg(reinterpret_cast<const double2*>(a));
        w[2 * i] = t.x;
        w[2 * i + 1] = t.y;
      } else {
        w[2 * i] = ok0(i, lim) ? __ldcg(a) : 0.0;
        w[2 * i + 1] = 0.0;
      }
    }
  };
  auto ov_store = [&](int q, const double (&w)[U]) {
    const int lim = len - q * E;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      double* a = wov + (int64_t)q * E + 2 * CT * i;
      if (lim >= E || ok1(i, lim)) __stcg(reinterpret_cast<double2*>(a), make_double2(w[2 * i], w[2 * i + 1]));
      else if (ok0(i, lim)) __stcg(a, w[2 * i]);
    }
  };
  auto ov_pass = [&](int kind, double& acc) {
    if (nch <= nrc) return;
    double cur[U], nxt[U];
    ov_load(nrc, cur);
#pragma unroll 1
    for (int q = nrc; q < nch; ++q) {
      if (q + 1 < nch) ov_load(q + 1, nxt);
      const int lim = len - q * E;
      const bool fullc = lim >= E;
      if (kind > 0) {   // w -= h_{p-1} V_{p-1}
        const double* sp = take();
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          Pair t = lds2(sp + 2 * CT * i);
          cur[2 * i] -= h * (fullc || ok0(i, lim) ? t.x : 0.0);
          cur[2 * i + 1] -= h * (fullc || ok1(i, lim) ? t.y : 0.0);
        }
        give();
      }
      if (kind < 2) {   // acc += V_p . w
        const double* sv = take();
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          Pair t = lds2(sv + 2 * CT * i);
          acc += (fullc || ok0(i, lim) ? t.x : 0.0) * cur[2 * i];
          acc += (fullc || ok1(i, lim) ? t.y : 0.0) * cur[2 * i + 1];
        }
        give();
      } else {          // acc += w . w
#pragma unroll
        for (int i = 0; i < U; ++i) acc += cur[i] * cur[i];
      }
      if (kind > 0) ov_store(q, cur);
#pragma unroll
      for (int i = 0; i < U; ++i) cur[i] = nxt[i];
    }
  };

  auto finish_pass = [&](int p, double acc) {
    t_wait_st();
    // CTA reduction (fixed order) then grid exchange
    acc = wsum(acc);
    if (lane == 0) scratch[warp] = acc;
    if (A.trace && threadIdx.x == 0) A.trace[((size_t)blockIdx.x * npass + p) * 4 + 1] = gtimer();
    named_sync(1, CT);
    if (warp == 0) {
      double c = lane < CW ? scratch[lane] : 0.0;
      c = wsum(c);
      if (A.trace && threadIdx.x == 0) A.trace[((size_t)blockIdx.x * npass + p) * 4 + 2] = gtimer();
      const double tot = grid_exchange(A, c, p);
      if (A.trace && threadIdx.x == 0) A.trace[((size_t)blockIdx.x * npass + p) * 4 + 3] = gtimer();
      if (lane == 0) scratch[32 + (p & 1)] = tot;
    }
    named_sync(1, CT);
    h = scratch[32 + (p & 1)];
    if (lead && p <= j) A.H[p * A.m + j] = h;
  };
  auto stamp = [&](int p) {
    if (A.trace && threadIdx.x == 0) A.trace[((size_t)blockIdx.x * npass + p) * 4 + 0] = gtimer();
  };
  // register-resident chunks of w (g is a compile-time constant in the unrolled loops)
#define WL_REG(k, i, wx, wy)              \
  {                                       \
    wx = wr[GQ * g + (k)][2 * (i)];       \
    wy = wr[GQ * g + (k)][2 * (i) + 1];   \
  }
#define WS_REG(k, i, wx, wy)              \
  {                                       \
    wr[GQ * g + (k)][2 * (i)] = (wx);     \
    wr[GQ * g + (k)][2 * (i) + 1] = (wy); \
  }
  // shared-memory chunks of w
#define WADDR(k, i) (wsm + (size_t)(GQ * g + (k) - RR) * E + e0 + 2 * CT * (i))
#define WL_SM(k, i, wx, wy)            \
  {                                    \
    const Pair t_ = lds2(WADDR(k, i)); \
    wx = t_.x;                         \
    wy = t_.y;                         \
  }
#define WS_SM(k, i, wx, wy) sts2(WADDR(k, i), (wx), (wy))
#define MGS_PASS(KIND)                                                            \
  {                                                                               \
    _Pragma("unroll") for (int g = 0; g < RR / GQ; ++g) if (GQ * g < nrc)          \
        MGS_GROUP(KIND, g, WL_REG, WS_REG)                                        \
    _Pragma("unroll 1") for (int g = RR / GQ; GQ * g < nrc; ++g)                   \
        MGS_GROUP(KIND, g, WL_SM, WS_SM)                                          \
    if constexpr (OV) ov_pass(KIND, acc);                                         \
  }
  {  // pass 0: stage w, h_0 = V_0 . w, V_0 -> TMEM
    const int p = 0;
    double acc = 0.0;
    stamp(p);
    MGS_PASS(0)
    finish_pass(p, acc);
  }
  for (int p = 1; p <= j; ++p) {  // w -= h_{p-1} V_{p-1}; h_p = V_p . w; V_p -> TMEM
    double acc = 0.0;
    stamp(p);
    MGS_PASS(1)
    finish_pass(p, acc);
  }
  {  // final: w -= h_j V_j; ||w||^2
    const int p = j + 1;
    double acc = 0.0;
    stamp(p);
    MGS_PASS(2)
    finish_pass(p, acc);
  }
#undef MGS_PASS
#undef WL_REG
#undef WS_REG
#undef WL_SM
#undef WS_SM
#undef WADDR
#undef MGS_GROUP

  // V[j+1] = w / hnext
  const double hnext = sqrt(h);
  double* wg = A.V + (int64_t)(j + 1) * A.ld + lo + e0;
  auto put_w = [&](int q, double wx, double wy, int i) {
    const int lim = len - q * E;
    double* d = wg + (int64_t)q * E + 2 * CT * i;
    if (lim >= E || ok1(i, lim)) {
      *reinterpret_cast<double2*>(d) = make_double2(wx / hnext, wy / hnext);
    } else if (ok0(i, lim)) {
      d[0] = wx / hnext;
    }
  };
#pragma unroll
  for (int q = 0; q < RR; ++q)
    if (q < nrc) {
#pragma unroll
      for (int i = 0; i < NP; ++i) put_w(q, wr[q][2 * i], wr[q][2 * i + 1], i);
    }
#pragma unroll 1
  for (int q = RR; q < nrc; ++q) {
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const Pair t = lds2(wsm + (size_t)(q - RR) * E + e0 + 2 * CT * i);
      put_w(q, t.x, t.y, i);
    }
  }
  if constexpr (OV) {
#pragma unroll 1
    for (int q = nrc; q < nch; ++q) {   // overflow: w is already in place in the V[j+1] row
      double w[U];
      ov_load(q, w);
#pragma unroll
      for (int i = 0; i < NP; ++i) put_w(q, w[2 * i], w[2 * i + 1], i);
    }
  }
  if (lead) givens(A, hnext);
  asm volatile("tcgen05.fence::before_thread_sync;");
  named_sync(1, CT);
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tbase), "n"(TCOLS));
  }
}

// host-side launch geometry for a slice of `chunk` elements; nres < the
// chunk count selects the partially resident (overflow) mode
inline bool plan(int64_t chunk, int* chunk_count, int* nsb, int* nres) {
  const int nch = (int)((chunk + E - 1) / E);
  if (nch > MAXCH_OV) return false;
  const bool ov = nch > MAXCH;
  const int res = ov ? MAXCH_RES_OV : nch;
  const int rr = ov ? R_OV : R;
  const int wch = res > rr ? res - rr : 0;
  const int64_t room = (int64_t)SMEM - HDR - (int64_t)wch * E * 8;
  int s = (int)(room / (E * 8));
  if (s > NSB_MAX) s = NSB_MAX;
  if (s < 2) return false;
  *chunk_count = nch;
  *nsb = s;
  *nres = res;
  return true;
}

}  // namespace mgs
}  // namespace svb
