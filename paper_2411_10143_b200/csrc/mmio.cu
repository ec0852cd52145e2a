// Matrix Market ingest on the B200 host + device.
//
// svb_mm_*: a multi-threaded parser of coordinate files with the reference's
// validation and messages (mmio.py:32-126): banner, object/format/field/
// symmetry, size line, per-entry field count, integer/float syntax, 1-based
// index range, more/fewer entries than declared — the error of the lowest
// failing entry wins, as in the sequential reference.
// svb_coo_from_triplets: CooMatrix.from_triplets (formats.py:86-100) on the
// device: stable radix sort of (row, col) keys, duplicates merged in
// np.add.reduceat order (p[s] + pairwise(p[s+1:e]), App. A.1).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "matrix.cuh"

struct svb_mm {
  std::string buf;
  size_t body = 0;  // first byte after the size line
  int64_t nrows = 0, ncols = 0, nnz = 0;
  bool pattern = false, symmetric = false;
};

namespace svb {
namespace {

constexpr int MM_ERROR = SVB_FORMAT_ERROR;

[[noreturn]] void fail(const std::string& msg) { throw Error{MM_ERROR, msg}; }

inline bool space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// [b, e) of the line starting at pos; returns the next line's start
inline size_t line_at(const std::string& s, size_t pos, size_t* b, size_t* e) {
  size_t nl = s.find('\n', pos);
  if (nl == std::string::npos) nl = s.size();
  *b = pos;
  *e = nl;
  return nl < s.size() ? nl + 1 : s.size();
}

inline void trim(const char*& b, const char*& e) {
  while (b < e && space(*b)) ++b;
  while (e > b && space(e[-1])) --e;
}

inline bool payload(const char* b, const char* e) {
  trim(b, e);
  return b < e && *b != '%';
}

std::vector<std::string> tokens(const char* b, const char* e) {
  std::vector<std::string> t;
  while (b < e) {
    while (b < e && space(*b)) ++b;
    const char* s = b;
    while (b < e && !space(*b)) ++b;
    if (b > s) t.emplace_back(s, b);
  }
  return t;
}

std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

// Python repr of a short ASCII line (for the "malformed fields" message)
std::string repr(const char* b, const char* e) {
  trim(b, e);
  std::string s(b, e);
  const bool sq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
  const char q = sq ? '"' : '\'';
  std::string out(1, q);
  for (char c : s) {
    if (c == '\\' || c == q) out += '\\';
    out += c;
  }
  out += q;
  return out;
}

inline bool parse_int(const char* b, const char* e, int64_t* v) {
  if (b < e && *b == '+') ++b;
  auto r = std::from_chars(b, e, *v);
  return r.ec == std::errc() && r.ptr == e;
}

inline bool parse_float(const char* b, const char* e, double* v) {
  if (b < e && *b == '+') ++b;
  auto r = std::from_chars(b, e, *v);
  if (r.ec == std::errc() && r.ptr == e) return true;
  if (r.ec == std::errc::result_out_of_range && r.ptr == e) {   // Python float(): +-inf / 0.0
    *v = strtod(std::string(b, e).c_str(), nullptr);
    return true;
  }
  return false;
}

struct ChunkOut {
  int64_t lines = 0;          // payload lines in the chunk
  int64_t err_k = -1;         // lowest failing entry index (global), -1 none
  std::string err;
};

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" {

int svb_mm_open(const char* path, int64_t* dims, int32_t* flags, svb_mm** out) {
  return guard([&] {
    SVB_REQUIRE(path && dims && flags && out, SVB_INVALID, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw Error{SVB_INVALID, std::string("cannot open ") + path};
    auto h = std::make_unique<svb_mm>();
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    h->buf.resize(sz > 0 ? (size_t)sz : 0);
    const size_t got = sz > 0 ? std::fread(&h->buf[0], 1, (size_t)sz, f) : 0;
    std::fclose(f);
    h->buf.resize(got);
    const std::string& s = h->buf;
    if (s.empty()) fail("empty input: missing banner");
    size_t b, e, pos = line_at(s, 0, &b, &e);
    {
      const char *lb = s.data() + b, *le = s.data() + e;
      auto head = tokens(lb, le);
      std::string trimmed(lb, le);
      const char* tb = trimmed.data();
      const char* te = tb + trimmed.size();
      trim(tb, te);
      if (head.size() != 5 || lower(head[0]) != "%%matrixmarket")
        fail("malformed banner: " + repr(tb, te));
      const std::string obj = lower(head[1]), fmt = lower(head[2]), fld = lower(head[3]), sym = lower(head[4]);
      if (obj != "matrix") fail("unsupported object '" + obj + "'");
      if (fmt != "coordinate") fail("unsupported format '" + fmt + "' (coordinate only)");
      if (fld == "complex") fail("complex matrices are not supported");
      if (fld != "real" && fld != "integer" && fld != "pattern") fail("unsupported field '" + fld + "'");
      if (sym != "general" && sym != "symmetric") fail("unsupported symmetry '" + sym + "'");
      h->pattern = fld == "pattern";
      h->symmetric = sym == "symmetric";
    }
    // size line: first payload line after the banner
    for (;;) {
      if (pos >= s.size()) fail("missing size line");
      pos = line_at(s, pos, &b, &e);
      if (payload(s.data() + b, s.data() + e)) break;
    }
    const char *lb = s.data() + b, *le = s.data() + e;
    trim(lb, le);
    auto t = tokens(lb, le);
    const std::string shown = repr(lb, le);
    if (t.size() != 3) fail("malformed size line: " + shown);
    int64_t v[3];
    for (int i = 0; i < 3; ++i)
      if (!parse_int(t[i].data(), t[i].data() + t[i].size(), &v[i])) fail("malformed size line: " + shown);
    if (v[0] < 1 || v[1] < 1 || v[2] < 0) fail("invalid dimensions in size line: " + shown);
    h->nrows = v[0];
    h->ncols = v[1];
    h->nnz = v[2];
    h->body = pos;
    dims[0] = h->nrows;
    dims[1] = h->ncols;
    dims[2] = h->nnz;
    flags[0] = h->pattern;
    flags[1] = h->symmetric;
    *out = h.release();
  });
}

int svb_mm_parse(svb_mm* h, int64_t* rows, int64_t* cols, double* vals, int32_t nthreads) {
  return guard([&] {
    SVB_REQUIRE(h, SVB_INVALID, "null handle");
    const std::string& s = h->buf;
    const size_t n0 = h->body, n1 = s.size();
    int T = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
    const size_t span = n1 > n0 ? n1 - n0 : 0;
    if ((size_t)T > span / (1 << 16) + 1) T = (int)(span / (1 << 16) + 1);   // >= 64 KB per thread
    // chunk bounds at line starts
    std::vector<size_t> cut(T + 1, n1);
    cut[0] = n0;
    for (int i = 1; i < T; ++i) {
      size_t p = n0 + span * i / T;
      if (p < cut[i - 1]) p = cut[i - 1];
      const size_t nl = s.find('\n', p > 0 ? p - 1 : 0);
      cut[i] = nl == std::string::npos ? n1 : nl + 1;
      if (cut[i] < cut[i - 1]) cut[i] = cut[i - 1];
    }
    std::vector<ChunkOut> res(T);
    auto run = [&](auto&& fn) {
      std::vector<std::thread> th;
      for (int i = 1; i < T; ++i) th.emplace_back(fn, i);
      fn(0);
      for (auto& t : th) t.join();
    };
    // pass 1: payload lines per chunk
    run([&](int i) {
      int64_t c = 0;
      size_t b, e;
      for (size_t pos = cut[i]; pos < cut[i + 1];) {
        pos = line_at(s, pos, &b, &e);
        if (e > cut[i + 1]) e = cut[i + 1];
        c += payload(s.data() + b, s.data() + e);
      }
      res[i].lines = c;
    });
    std::vector<int64_t> first(T + 1, 0);
    for (int i = 0; i < T; ++i) first[i + 1] = first[i] + res[i].lines;
    const int64_t total = first[T], nnz = h->nnz, nr = h->nrows, nc = h->ncols;
    const int want = h->pattern ? 2 : 3;
    // pass 2: parse entries with index < nnz, record the first failure
    run([&](int i) {
      int64_t k = first[i];
      size_t b, e;
      for (size_t pos = cut[i]; pos < cut[i + 1] && k < nnz;) {
        pos = line_at(s, pos, &b, &e);
        const char *lb = s.data() + b, *le = s.data() + e;
        if (!payload(lb, le)) continue;
        trim(lb, le);
        const char* f[3];
        const char* fe[3];
        int nf = 0;
        for (const char* p = lb; p < le;) {
          while (p < le && space(*p)) ++p;
          if (p >= le) break;
          const char* q = p;
          while (q < le && !space(*q)) ++q;
          if (nf < 3) {
            f[nf] = p;
            fe[nf] = q;
          }
          ++nf;
          p = q;
        }
        auto bad = [&](const std::string& m) {
          res[i].err_k = k;
          res[i].err = m;
        };
        if (nf != want) {
          bad("entry " + std::to_string(k + 1) + ": expected " + std::to_string(want) + " fields, got " +
              std::to_string(nf));
          return;
        }
        int64_t r, c;
        double v = 1.0;
        if (!parse_int(f[0], fe[0], &r) || !parse_int(f[1], fe[1], &c) ||
            (!h->pattern && !parse_float(f[2], fe[2], &v))) {
          bad("entry " + std::to_string(k + 1) + ": malformed fields " + repr(lb, le));
          return;
        }
        if (!(1 <= r && r <= nr && 1 <= c && c <= nc)) {
          bad("entry " + std::to_string(k + 1) + ": index (" + std::to_string(r) + ", " + std::to_string(c) +
              ") out of range for " + std::to_string(nr) + "x" + std::to_string(nc));
          return;
        }
        rows[k] = r - 1;
        cols[k] = c - 1;
        vals[k] = v;
        ++k;
      }
    });
    for (int i = 0; i < T; ++i)
      if (res[i].err_k >= 0) fail(res[i].err);   // chunks are in entry order: the first is the lowest
    if (total > nnz) fail("more entries than declared in size line");
    if (total < nnz) fail("truncated entries: got " + std::to_string(total) + ", expected " + std::to_string(nnz));
  });
}

int svb_mm_close(svb_mm* h) {
  return guard([&] { delete h; });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// from_triplets on the device
// ---------------------------------------------------------------------------
namespace svb {

__global__ void k_keys(int64_t n, const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t ncols,
                       unsigned long long* __restrict__ key, int64_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = (unsigned long long)(r[i] * ncols + c[i]);
    idx[i] = i;
  }
}

// run heads of the sorted keys (1 where a new (row, col) starts)
__global__ void k_heads(int64_t n, const unsigned long long* __restrict__ key, int64_t* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// one thread per run: rows/cols from the key, value = reduceat order over
// the run's values in input order (the sort is stable)
__global__ void k_runs(int64_t n, int64_t nruns, const int64_t* __restrict__ pos, const unsigned long long* __restrict__ key,
                       const int64_t* __restrict__ idx, const double* __restrict__ v, int64_t ncols,
                       int* __restrict__ rows, int* __restrict__ cols, double* __restrict__ out, bool merge) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool h = i == 0 || key[i] != key[i - 1];
    if (!merge) {
      rows[i] = (int)(key[i] / (unsigned long long)ncols);
      cols[i] = (int)(key[i] % (unsigned long long)ncols);
      out[i] = v[idx[i]];
      continue;
    }
    if (!h) continue;
    int64_t e = i + 1;
    while (e < n && key[e] == key[i]) ++e;
    const int64_t o = pos[i];
    rows[o] = (int)(key[i] / (unsigned long long)ncols);
    cols[o] = (int)(key[i] % (unsigned long long)ncols);
    out[o] = segment_sum<double>([&](int64_t k) { return v[idx[k]]; }, i, e);
  }
  (void)nruns;
}

}  // namespace svb

extern "C" int svb_coo_from_triplets(int64_t nrows, int64_t ncols, int64_t n, const int64_t* rows_host,
                                     const int64_t* cols_host, const double* vals_host, int32_t sum_duplicates,
                                     void* stream, svb_matrix** out) {
  return guard([&] {
    SVB_REQUIRE(nrows >= 1 && ncols >= 1 && n >= 0, SVB_INVALID, "matrix dimensions must be positive");
    SVB_REQUIRE(nrows < INT32_MAX && ncols < INT32_MAX, SVB_INAPPLICABLE,
                "dimensions exceed the int32 index range of the device layout");
    SVB_REQUIRE((double)nrows * (double)ncols < 9.0e18, SVB_INAPPLICABLE, "row*col key exceeds 63 bits");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto m = new svb_matrix();
    std::unique_ptr<svb_matrix> guard_m(m);
    m->fmt = SVB_COO;
    m->nrows = nrows;
    m->ncols = ncols;
    if (n == 0) {
      m->nnz = 0;
      m->rows = alloc(16, s);
      m->cols = alloc(16, s);
      m->vals = alloc(16, s);
      SVB_CUDA_TRY(cudaStreamSynchronize(s));
      *out = publish(guard_m.release());
      return;
    }
    Buf r = upload(rows_host, n * 8, s), c = upload(cols_host, n * 8, s), v = upload(vals_host, n * 8, s);
    Buf k0 = alloc(n * 8, s), k1 = alloc(n * 8, s), i0 = alloc(n * 8, s), i1 = alloc(n * 8, s);
    const unsigned g = grid_for(n, 256);
    k_keys<<<g, 256, 0, s>>>(n, ptr<int64_t>(r), ptr<int64_t>(c), ncols, ptr<unsigned long long>(k0),
                             ptr<int64_t>(i0));
    SVB_CHECK_LAUNCH();
    int bits = 1;
    while (bits < 64 && (((unsigned long long)nrows * (unsigned long long)ncols - 1) >> bits)) ++bits;
    size_t tmp_bytes = 0;
    SVB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ptr<unsigned long long>(k0),
                                                 ptr<unsigned long long>(k1), ptr<int64_t>(i0), ptr<int64_t>(i1),
                                                 n, 0, bits, s));
    Buf tmp = alloc(tmp_bytes + 16, s);
    SVB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp->ptr, tmp_bytes, ptr<unsigned long long>(k0),
                                                 ptr<unsigned long long>(k1), ptr<int64_t>(i0), ptr<int64_t>(i1),
                                                 n, 0, bits, s));
    Buf head = alloc((n + 1) * 8, s), pos = alloc((n + 1) * 8, s);
    int64_t nruns = n;
    if (sum_duplicates) {
      k_heads<<<g, 256, 0, s>>>(n, ptr<unsigned long long>(k1), ptr<int64_t>(head));
      SVB_CHECK_LAUNCH();
      nruns = exclusive_scan_total(ptr<int64_t>(head), ptr<int64_t>(pos), n, s);
    }
    m->nnz = nruns;
    m->ptr64 = want_ptr64(nruns);
    m->rows = alloc(nruns * 4, s);
    m->cols = alloc(nruns * 4, s);
    m->vals = alloc(nruns * 8, s);
    k_runs<<<g, 256, 0, s>>>(n, nruns, ptr<int64_t>(pos), ptr<unsigned long long>(k1), ptr<int64_t>(i1),
                             ptr<double>(v), ncols, ptr<int>(m->rows), ptr<int>(m->cols), ptr<double>(m->vals),
                             sum_duplicates != 0);
    SVB_CHECK_LAUNCH();
    SVB_CUDA_TRY(cudaStreamSynchronize(s));
    *out = publish(guard_m.release());
  });
}
