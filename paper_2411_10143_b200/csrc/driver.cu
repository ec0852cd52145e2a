// Native solver drivers and the configuration mailbox (SURVEY.md §8b:
// "device-resident solver drivers ... with mailbox hooks").
//
// svb_gmres_run / svb_cg_run are the host loops of the Python drivers
// (paper_2411_10143_b200/solver.py _gmres_core / _cg_core, which restate
// the reference's _gmres_core, solver.py:219-342, and the new CG) in C++, for
// hosts that bind the C ABI without Python (cgo, JNI, a C++ service).  They
// enqueue the same kernels in the same order as the Python loops, so reports
// and solutions are bit-identical to gmres_solve / cg_solve with the same
// configuration:
//   * GMRES: one SpMV + one fused Arnoldi kernel per step; the next step's
//     normalisation and SpMV are enqueued before the host reads the step's
//     status (speculation: discarded if the loop exits, restarts or swaps);
//   * CG: batches of 1, 2, 4, ... 32 iterations with no host read inside a
//     batch (kernels after the converging iteration are no-ops), full
//     batches replayed as CUDA graphs, DIA operators through the fused
//     SpMV + p.q step.
// The mailbox (ConfigMailbox, solver.py:126-185) is last-writer-wins: any
// host thread (the advisor) publishes a matrix handle in the configuration's
// format plus an optional event the handle is complete at; the driver polls
// between iterations, and a different configuration is swapped in for the
// next iteration and recorded in the timeline.
#include <cmath>
#include <cstdio>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

struct svb_mailbox {
  std::mutex mu;
  bool pending = false;
  const svb_matrix* m = nullptr;
  svb_config cfg{};
  void* ready = nullptr;
  double prep = 0.0;
  bool finished = false;
};

namespace {

using svb::Error;

void ck(int status) {
  if (status != SVB_OK) throw Error{status, svb::get_error()};
}

bool same_config(const svb_config& a, const svb_config& b) {
  // SpmvConfig equality (kernels.py:44-86): workers is a run-time argument,
  // not part of the configuration
  return a.format == b.format && a.library == b.library && a.lane == b.lane;
}

void check_finite(double v, const char* what, int iteration) {
  if (!std::isfinite(v)) {
    char buf[160];
    snprintf(buf, sizeof buf, "non-finite %s at iteration %d; aborting", what, iteration);
    throw Error{SVB_NONFINITE, buf};
  }
}

// Workspaces are recycled across solves (as solver.py's _acquire_ws): a
// fresh one would cost a 1 GB allocation at config 2 and the device-wide
// synchronisation of svb_krylov_destroy.
std::mutex g_pool_mu;
struct Pooled {
  int64_t n;
  int m;
  svb_krylov* k;
};
std::vector<Pooled> g_pool;
constexpr size_t POOL_KEEP = 2;

svb_krylov* acquire_ws(int64_t n, int m) {
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    for (size_t i = 0; i < g_pool.size(); ++i)
      if (g_pool[i].n == n && g_pool[i].m == m) {
        svb_krylov* k = g_pool[i].k;
        g_pool.erase(g_pool.begin() + i);
        return k;
      }
  }
  svb_krylov* k = nullptr;
  ck(svb_krylov_create(n, m, &k));
  return k;
}
void release_ws(int64_t n, int m, svb_krylov* k, void* stream) {
  cudaStreamSynchronize((cudaStream_t)stream);   // nothing of this solve still in flight
  std::lock_guard<std::mutex> g(g_pool_mu);
  g_pool.push_back({n, m, k});
  if (g_pool.size() > POOL_KEEP) {
    svb_krylov* old = g_pool.front().k;
    g_pool.erase(g_pool.begin());
    svb_krylov_destroy(old);
  }
}

struct Run {
  const svb_matrix* A = nullptr;
  svb_config cfg{};
  svb_mailbox* mb = nullptr;
  void* s = nullptr;
  svb_krylov* k = nullptr;
  double* hist = nullptr;
  int hist_cap = 0;
  svb_swap* tl = nullptr;
  int tl_cap = 0;
  svb_solve_report* rep = nullptr;
  int completed = 0;
  int version = 0;   // bumps on every swap (speculation validity)
  int m_ = 0;

  ~Run() {   // also on the error paths: the advisor may stop, the workspace is recycled
    if (k) release_ws(n_, m_, k, s);
    if (mb) {
      std::lock_guard<std::mutex> g(mb->mu);
      mb->finished = true;
    }
  }
  double* vec(int which) {
    double* p = nullptr;
    ck(svb_krylov_vec(k, which, &p));
    return p;
  }
  svb_krylov_status status() {
    svb_krylov_status st;
    ck(svb_krylov_status_get(k, s, &st));
    return st;
  }
  void spmv(const double* x, double* y) {
    ck(svb_spmv(A, cfg.format, cfg.library, cfg.lane, cfg.workers, SVB_F64, x, y, s));
  }
  void record(double est) {
    if (rep->history_len < hist_cap) hist[rep->history_len] = est;
    rep->history_len++;
  }
  void add_swap(int iteration, const svb_config& c, double prep) {
    if (rep->nswaps < tl_cap) {
      tl[rep->nswaps].iteration = iteration;
      tl[rep->nswaps].config = c;
      tl[rep->nswaps].prep_seconds = prep;
    }
    rep->nswaps++;
  }
  // ConfigMailbox.poll + _swap_handler (solver.py:410-421)
  void poll() {
    if (!mb) return;
    const svb_matrix* m;
    svb_config c;
    void* ready;
    double prep;
    {
      std::lock_guard<std::mutex> g(mb->mu);
      if (!mb->pending) return;
      mb->pending = false;
      m = mb->m;
      c = mb->cfg;
      ready = mb->ready;
      prep = mb->prep;
    }
    if (!m || same_config(c, cfg)) return;
    if (ready) ck(svb_stream_wait_event(s, ready));
    A = m;
    cfg = c;
    version++;
    add_swap(completed + 1, c, prep);
  }
  double true_residual(double bnorm) {
    spmv(vec(-1), vec(-3));
    ck(svb_krylov_residual(k, s));
    return status().beta / bnorm;
  }
  void finish(bool converged, double final_res, double* x_dev) {
    SVB_CUDA_TRY(cudaMemcpyAsync(x_dev, vec(-1), (size_t)svb_n() * 8, cudaMemcpyDeviceToDevice,
                                 (cudaStream_t)s));
    SVB_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)s));
    rep->converged = converged;
    rep->iterations = completed;
    rep->final_residual = final_res;
    if (mb) {
      std::lock_guard<std::mutex> g(mb->mu);
      mb->finished = true;
    }
  }
  int64_t n_ = 0;
  int64_t svb_n() const { return n_; }
};

void start(Run& r, const svb_matrix* A, svb_config cfg, const double* b_dev, const svb_solve_params* p,
           int m, svb_mailbox* mb, void* stream, double* hist, svb_swap* tl, int32_t tl_cap,
           svb_solve_report* rep, const char* method) {
  SVB_REQUIRE(A && b_dev && p && rep && (hist || p->max_iters == 0), SVB_INVALID,
              "svb_*_run: null argument");
  SVB_REQUIRE(p->max_iters >= 0 && p->tol >= 0.0, SVB_INVALID, "max_iters and tol must be non-negative");
  svb_matrix_info info;
  ck(svb_matrix_info_get(A, &info));
  if (info.nrows != info.ncols) {
    throw Error{SVB_DIM_MISMATCH, std::string(method) + " requires a square matrix matching b"};
  }
  r.A = A;
  r.cfg = cfg;
  r.mb = mb;
  r.s = stream;
  r.hist = hist;
  r.hist_cap = p->max_iters > 0 ? p->max_iters : 0;
  r.tl = tl;
  r.tl_cap = tl ? tl_cap : 0;
  r.rep = rep;
  r.n_ = info.nrows;
  r.m_ = m;
  *rep = svb_solve_report{};
  rep->final_residual = NAN;
  if (mb) {
    std::lock_guard<std::mutex> g(mb->mu);
    mb->finished = false;
  }
  r.k = acquire_ws(info.nrows, m);
  SVB_CUDA_TRY(cudaMemcpyAsync(r.vec(-2), b_dev, (size_t)info.nrows * 8, cudaMemcpyDeviceToDevice,
                               (cudaStream_t)stream));
  SVB_CUDA_TRY(cudaMemsetAsync(r.vec(-1), 0, (size_t)info.nrows * 8, (cudaStream_t)stream));
  r.add_swap(1, cfg, 0.0);
}

constexpr int CG_BATCH = 32;

}  // namespace

extern "C" {

int svb_mailbox_create(svb_mailbox** out) {
  return svb::guard([&] { *out = new svb_mailbox(); });
}
int svb_mailbox_destroy(svb_mailbox* mb) {
  return svb::guard([&] { delete mb; });
}
int svb_mailbox_publish(svb_mailbox* mb, const svb_matrix* m, svb_config cfg, void* ready_event,
                        double prep_seconds) {
  return svb::guard([&] {
    SVB_REQUIRE(mb, SVB_INVALID, "null mailbox");
    std::lock_guard<std::mutex> g(mb->mu);
    mb->pending = true;
    mb->m = m;
    mb->cfg = cfg;
    mb->ready = ready_event;
    mb->prep = prep_seconds;
  });
}
int svb_mailbox_finished(svb_mailbox* mb, int32_t* out) {
  return svb::guard([&] {
    SVB_REQUIRE(mb && out, SVB_INVALID, "null argument");
    std::lock_guard<std::mutex> g(mb->mu);
    *out = mb->finished;
  });
}

// _gmres_core (solver.py:424-517)
int svb_gmres_run(const svb_matrix* A, svb_config cfg, const double* b_dev, double* x_dev,
                  const svb_solve_params* p, svb_mailbox* mb, void* stream, double* history_host,
                  svb_swap* timeline_host, int32_t timeline_cap, svb_solve_report* out) {
  return svb::guard([&] {
    SVB_REQUIRE(p && p->restart_m >= 1, SVB_INVALID, "restart_m must be >= 1");
    Run r;
    const int m = p->restart_m;
    start(r, A, cfg, b_dev, p, m, mb, stream, history_host, timeline_host, timeline_cap, out, "GMRES");
    ck(svb_krylov_bnorm(r.k, stream));
    const double bnorm = r.status().beta;
    if (bnorm == 0.0) {
      if (p->max_iters >= 1) r.record(0.0);
      r.finish(true, 0.0, x_dev);
      return;
    }
    if (p->max_iters == 0) {
      r.finish(false, NAN, x_dev);
      return;
    }
    int spec_src = -100, spec_ver = -1;   // speculative SpMV V[j+1] -> V[j+2] enqueued
    auto op = [&](int src, int dst) {
      if (spec_src == src && spec_ver == r.version) {
        spec_src = -100;
        return;
      }
      spec_src = -100;
      r.spmv(r.vec(src), r.vec(dst));
    };
    auto& done = r.completed;
    while (done < p->max_iters) {
      spec_src = -100;
      r.spmv(r.vec(-1), r.vec(-3));
      ck(svb_gmres_restart(r.k, stream));
      const double beta = r.status().beta;
      check_finite(beta, "residual norm", done);
      if (beta / bnorm <= p->tol) {
        r.finish(true, beta / bnorm, x_dev);
        return;
      }
      bool applied = false;
      int j = -1;   // as Python's loop variable: the last step run (-1: none)
      for (int jj = 0; jj < m; ++jj) {
        if (done >= p->max_iters) break;
        j = jj;
        op(j, j + 1);
        ck(svb_gmres_arnoldi(r.k, j, bnorm, stream));
        if (j + 1 < m && done + 1 < p->max_iters) {
          ck(svb_gmres_normalize(r.k, j, stream));
          r.spmv(r.vec(j + 1), r.vec(j + 2));
          spec_src = j + 1;
          spec_ver = r.version;
        }
        const svb_krylov_status st = r.status();
        check_finite(st.hnext, "Arnoldi norm", done + 1);
        ++done;
        check_finite(st.estimate, "residual estimate", done);
        r.record(st.estimate);
        if (st.hnext == 0.0) {
          if (st.hjj != 0.0) ck(svb_gmres_update_x(r.k, j, stream));
          const double fin = r.true_residual(bnorm);
          r.finish(fin <= p->tol, fin, x_dev);
          out->stagnated = !(fin <= p->tol);
          return;
        }
        if (st.estimate <= p->tol) {
          ck(svb_gmres_update_x(r.k, j, stream));
          const double fin = r.true_residual(bnorm);
          if (fin <= p->tol) {
            r.finish(true, fin, x_dev);
            return;
          }
          applied = true;   // estimate drifted: restart from x
          r.poll();
          break;
        }
        r.poll();
        ck(svb_gmres_normalize(r.k, j, stream));
      }
      if (j >= 0 && !applied) ck(svb_gmres_update_x(r.k, j, stream));
    }
    const double fin = r.true_residual(bnorm);
    r.finish(fin <= p->tol, fin, x_dev);
  });
}

// _cg_core, batched path (solver.py:520-645)
int svb_cg_run(const svb_matrix* A, svb_config cfg, const double* b_dev, double* x_dev,
               const svb_solve_params* p, svb_mailbox* mb, void* stream, double* history_host,
               svb_swap* timeline_host, int32_t timeline_cap, svb_solve_report* out) {
  return svb::guard([&] {
    Run r;
    start(r, A, cfg, b_dev, p, 0, mb, stream, history_host, timeline_host, timeline_cap, out, "CG");
    ck(svb_krylov_bnorm(r.k, stream));
    const double bnorm = r.status().beta;
    if (bnorm == 0.0) {
      if (p->max_iters >= 1) r.record(0.0);
      r.finish(true, 0.0, x_dev);
      return;
    }
    if (p->max_iters == 0) {
      r.finish(false, NAN, x_dev);
      return;
    }
    SVB_CUDA_TRY(cudaMemsetAsync(r.vec(-3), 0, (size_t)r.n_ * 8, (cudaStream_t)stream));   // A x0, x0 = 0
    ck(svb_cg_restart(r.k, stream));
    ck(svb_cg_batch_reset(r.k, p->tol, p->max_iters > 1 ? p->max_iters : 1, stream));
    double* P = r.vec(-4);
    double* Q = r.vec(-5);
    // one graph per (operator, configuration), built after one uncaptured
    // batch of that operator (lazily built per-matrix state never gets
    // created inside a capture)
    struct G {
      const svb_matrix* a;
      svb_config c;
      void* exec;
    };
    std::vector<G> graphs;
    std::vector<std::pair<const svb_matrix*, svb_config>> warm;
    auto enqueue = [&](int nb) {
      for (int t = 0; t < nb; ++t) {
        if (r.cfg.format == SVB_DIA) {
          ck(svb_cg_step_batched_dia(r.k, r.A, bnorm, stream));
        } else {
          r.spmv(P, Q);
          ck(svb_cg_step_batched(r.k, bnorm, stream));
        }
      }
    };
    auto is_warm = [&]() {
      for (auto& e : warm)
        if (e.first == r.A && same_config(e.second, r.cfg)) return true;
      return false;
    };
    auto find_graph = [&]() -> G* {
      for (auto& e : graphs)
        if (e.a == r.A && same_config(e.c, r.cfg)) return &e;
      return nullptr;
    };
    auto run_batch = [&](int nb) {
      if (nb != CG_BATCH || !is_warm()) {
        enqueue(nb);
        if (!is_warm()) warm.push_back({r.A, r.cfg});
        return;
      }
      G* g = find_graph();
      if (!g) {
        void* exec = nullptr;
        ck(svb_graph_begin(stream));
        try {
          enqueue(nb);
        } catch (...) {
          svb_graph_end(stream, &exec);
          if (exec) svb_graph_destroy(exec);
          throw;
        }
        ck(svb_graph_end(stream, &exec));
        graphs.push_back({r.A, r.cfg, exec});
        g = &graphs.back();
      }
      ck(svb_graph_launch(g->exec, stream));
      ck(svb_krylov_mark(r.k, stream));
    };
    auto cleanup = [&] {
      if (!graphs.empty()) {
        cudaStreamSynchronize((cudaStream_t)stream);
        for (auto& g : graphs) svb_graph_destroy(g.exec);
        graphs.clear();
      }
    };
    try {
      int64_t base = 0;
      int batch = 1;
      auto& done = r.completed;
      std::vector<double> est;
      bool returned = false;
      while (done < p->max_iters) {
        const int nb = batch < p->max_iters - done ? batch : p->max_iters - done;
        run_batch(nb);
        batch = batch * 2 < CG_BATCH ? batch * 2 : CG_BATCH;
        const svb_krylov_status st = r.status();
        const int64_t ran = st.count - base;
        est.resize(ran > 0 ? ran : 0);
        if (ran > 0) ck(svb_cg_history(r.k, base, ran, est.data(), stream));
        base += ran;
        for (int64_t t = 0; t < ran; ++t) check_finite(est[t], "residual estimate", done + (int)t + 1);
        for (int64_t t = 0; t < ran; ++t) r.record(est[t]);
        done += (int)ran;
        if (st.done == 3) {
          check_finite(st.pq, "curvature p.Ap", done + 1);
          check_finite(NAN, "residual estimate", done);
        }
        if (st.done == 2) {   // p.Ap == 0: breakdown
          const double fin = r.true_residual(bnorm);
          r.finish(fin <= p->tol, fin, x_dev);
          out->stagnated = !(fin <= p->tol);
          returned = true;
          break;
        }
        if (st.done == 1) {
          const double fin = r.true_residual(bnorm);
          if (fin <= p->tol) {
            r.finish(true, fin, x_dev);
            returned = true;
            break;
          }
          ck(svb_cg_restart(r.k, stream));   // r = b - A x, p = r
          ck(svb_cg_batch_resume(r.k, stream));
          continue;
        }
        r.poll();
      }
      if (!returned) {
        const double fin = r.true_residual(bnorm);
        r.finish(fin <= p->tol, fin, x_dev);
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

}  // extern "C"
