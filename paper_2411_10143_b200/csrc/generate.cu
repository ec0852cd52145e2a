// On-device CSR generation for constant-coefficient stencils on Cartesian
// grids (BASELINE.json configs 1, 2 and 5).  Config 5 (600^3, 5.8e9 nnz)
// cannot be staged through host memory, so the matrix is built where it is
// used.  Output is identical to generators.stencil_csr on the host: rows in
// grid order (fastest axis last), columns ascending, out-of-grid neighbours
// dropped.
#include <algorithm>
#include <numeric>
#include <vector>

#include "matrix.cuh"

namespace svb {

constexpr int MAX_DIM = 4;
constexpr int MAX_ST = 128;

struct Stencil {
  int ndim, nst;
  int64_t dims[MAX_DIM];
  int off[MAX_ST][MAX_DIM];
  int64_t lin[MAX_ST];
  double w[MAX_ST];
};

__device__ __forceinline__ void coords_of(const Stencil& st, int64_t i, int64_t* c) {
  for (int a = st.ndim - 1; a >= 0; --a) {
    c[a] = i % st.dims[a];
    i /= st.dims[a];
  }
}

__device__ __forceinline__ bool inside(const Stencil& st, const int64_t* c, int s) {
  for (int a = 0; a < st.ndim; ++a) {
    const int64_t v = c[a] + st.off[s][a];
    if (v < 0 || v >= st.dims[a]) return false;
  }
  return true;
}

// rows [r0, r0 + n) of the global stencil matrix
__global__ void k_stencil_count(Stencil st, int64_t n, int64_t r0, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[MAX_DIM];
    coords_of(st, r0 + i, c);
    int64_t k = 0;
    for (int s = 0; s < st.nst; ++s) k += inside(st, c, s);
    cnt[i] = k;
  }
}

// columns stored relative to `cmin` (a row block's column window)
__global__ void k_stencil_fill(Stencil st, int64_t n, int64_t r0, int64_t cmin, const int64_t* __restrict__ ptr,
                               int* __restrict__ cols, double* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[MAX_DIM];
    coords_of(st, r0 + i, c);
    int64_t o = ptr[i];
    for (int s = 0; s < st.nst; ++s) {
      if (!inside(st, c, s)) continue;
      cols[o] = (int)(r0 + i + st.lin[s] - cmin);
      vals[o] = st.w[s];
      ++o;
    }
  }
}

}  // namespace svb

using namespace svb;

static svb_matrix* stencil_rows(int ndim, const int64_t* dims, int nst, const int32_t* offsets,
                                const double* weights, int64_t r0, int64_t r1, int64_t cmin, int64_t ncols,
                                cudaStream_t s) {
  SVB_REQUIRE(ndim >= 1 && ndim <= MAX_DIM && nst >= 1 && nst <= MAX_ST, SVB_INVALID,
              "stencil: 1..4 dimensions, 1..128 points");
  Stencil st{};
  st.ndim = ndim;
  st.nst = nst;
  int64_t N = 1;
  for (int a = 0; a < ndim; ++a) {
    SVB_REQUIRE(dims[a] >= 1, SVB_INVALID, "stencil: grid dimensions must be positive");
    st.dims[a] = dims[a];
    N *= dims[a];
  }
  SVB_REQUIRE(0 <= r0 && r0 < r1 && r1 <= N, SVB_INVALID, "stencil: bad row range");
  SVB_REQUIRE(ncols < INT32_MAX, SVB_INAPPLICABLE, "stencil column window exceeds the int32 index range");
  std::vector<int64_t> lin(nst);
  for (int k = 0; k < nst; ++k) {
    int64_t l = 0, stride = 1;
    for (int a = ndim - 1; a >= 0; --a) {
      l += (int64_t)offsets[k * ndim + a] * stride;
      stride *= dims[a];
    }
    lin[k] = l;
  }
  std::vector<int> order(nst);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return lin[a] < lin[b]; });
  for (int k = 0; k < nst; ++k) {
    const int src = order[k];
    for (int a = 0; a < ndim; ++a) st.off[k][a] = offsets[src * ndim + a];
    st.lin[k] = lin[src];
    st.w[k] = weights[src];
  }
  const int64_t n = r1 - r0;
  Buf cnt = alloc(n * 8, s);
  k_stencil_count<<<grid_for(n, 256), 256, 0, s>>>(st, n, r0, ptr<int64_t>(cnt));
  SVB_CHECK_LAUNCH();
  Buf ptr64 = alloc((n + 1) * 8, s);
  const int64_t nnz = exclusive_scan_total(ptr<int64_t>(cnt), ptr<int64_t>(ptr64), n, s);
  cnt.reset();
  auto m = new svb_matrix();
  m->fmt = SVB_CSR;
  m->nrows = n;
  m->ncols = ncols;
  m->nnz = nnz;
  m->ptr64 = want_ptr64(nnz);
  m->cols = alloc(nnz * 4, s);
  m->vals = alloc(nnz * 8, s);
  k_stencil_fill<<<grid_for(n, 256), 256, 0, s>>>(st, n, r0, cmin, ptr<int64_t>(ptr64), ptr<int>(m->cols),
                                                 ptr<double>(m->vals));
  SVB_CHECK_LAUNCH();
  if (m->ptr64) m->ptr = ptr64;
  else {
    m->ptr = alloc((n + 1) * 4, s);
    narrow_i64_to_i32(ptr<int64_t>(ptr64), ptr<int32_t>(m->ptr), n + 1, s);
  }
  SVB_CUDA_TRY(cudaStreamSynchronize(s));
  return publish(m);
}

extern "C" int svb_csr_stencil(int ndim, const int64_t* dims, int nst, const int32_t* offsets,
                               const double* weights, void* stream, svb_matrix** out) {
  return guard([&] {
    int64_t n = 1;
    for (int a = 0; a < ndim && a < MAX_DIM; ++a) n *= dims[a] > 0 ? dims[a] : 1;
    SVB_REQUIRE(n < INT32_MAX, SVB_INAPPLICABLE, "stencil grid exceeds the int32 column index range");
    *out = stencil_rows(ndim, dims, nst, offsets, weights, 0, n, 0, n, reinterpret_cast<cudaStream_t>(stream));
  });
}

extern "C" int svb_csr_stencil_rows(int ndim, const int64_t* dims, int nst, const int32_t* offsets,
                                    const double* weights, int64_t r0, int64_t r1, int64_t cmin, int64_t cmax,
                                    void* stream, svb_matrix** out) {
  return guard([&] {
    SVB_REQUIRE(cmin <= r0 && cmax >= r1 - 1 && cmin >= 0, SVB_INVALID,
                "stencil block: the column window must cover the block's own rows");
    *out = stencil_rows(ndim, dims, nst, offsets, weights, r0, r1, cmin, cmax - cmin + 1,
                        reinterpret_cast<cudaStream_t>(stream));
  });
}
