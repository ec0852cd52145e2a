"""CPU reference timing for bench.py — TEST/MEASUREMENT INFRASTRUCTURE ONLY.

Times the reference algorithm (this package's numpy restatement, pinned
bit-exact to /root/reference by tests/test_oracle_golden.py) on the GPU
box's host cores, for the bench workload: the reference's predict-then-solve
flow (solver.py:496-540) — features -> cascade (shipped models) -> format
conversion -> restarted GMRES — on the 9-point convection-diffusion matrix.

A full CPU solve takes ~30 s, so each sample runs the whole
preprocessing plus ``iters`` GMRES iterations at full size and extrapolates
the solve to ``total_iters`` iterations (stated in the output "sample").

    python -m oracle.bench_cpu --nx 2000 --iters 4 --total-iters 77 --repeat 1
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

from . import cpu_oracle as O

ROOT = Path(__file__).resolve().parent.parent


def convdiff9_csr(nx: int, diag: float = 8.5, beta: float = 0.25) -> O.OCsr:
    """Same structure as paper_2411_10143_b200.generators.convdiff9 (restated
    here so the oracle never imports the product)."""
    n = nx * nx
    y, x = np.divmod(np.arange(n, dtype=np.int64), nx)
    cols, vals, masks = [], [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            ok = (x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < nx)
            masks.append(ok)
            cols.append(np.arange(n, dtype=np.int64) + dy * nx + dx)
            vals.append(diag if (dx, dy) == (0, 0) else -1.0 - beta * (dx + dy))
    masks = np.stack(masks)
    lens = masks.sum(axis=0)
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    c2 = np.stack(cols)
    v2 = np.broadcast_to(np.asarray(vals)[:, None], masks.shape)
    return O.OCsr(n, n, ptr, c2.T[masks.T], np.ascontiguousarray(v2.T[masks.T]))


def laplace27_csr(n3: int) -> O.OCsr:
    """3-D 27-point Laplacian n3^3 (diag 26, off -1), same structure as
    paper_2411_10143_b200.generators.laplace27 (restated: the oracle never
    imports the product)."""
    n = n3 ** 3
    z, rem = np.divmod(np.arange(n, dtype=np.int64), n3 * n3)
    y, x = np.divmod(rem, n3)
    cols, vals, masks = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                masks.append((x + dx >= 0) & (x + dx < n3) & (y + dy >= 0) & (y + dy < n3) &
                             (z + dz >= 0) & (z + dz < n3))
                cols.append(np.arange(n, dtype=np.int64) + (dz * n3 + dy) * n3 + dx)
                vals.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
    masks = np.stack(masks)
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(masks.sum(axis=0), out=ptr[1:])
    c2 = np.stack(cols)
    v2 = np.broadcast_to(np.asarray(vals)[:, None], masks.shape)
    return O.OCsr(n, n, ptr, c2.T[masks.T], np.ascontiguousarray(v2.T[masks.T]))


def cg_sample(n3: int, iters: int, total_iters: int, target_n3: int, models) -> dict:
    """Config 5 on the CPU: the reference's predict-then-solve with the new CG
    oracle on a n3^3 grid, `iters` CG iterations timed; preprocessing and the
    per-iteration time are scaled per nnz to target_n3^3 and the solve to
    total_iters iterations (the full 600^3 matrix does not fit the host)."""
    csr = laplace27_csr(n3)
    b = O.spmv_sequential(csr, np.ones(csr.nrows))
    t = {}
    t0 = time.perf_counter()
    coo = O.csr_to_coo(csr)
    fv = O.features(O.coo_to_csr(coo))
    t["features"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    final = O.cascade(models, fv)[-1]
    t["inference"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rep = O.convert(coo, final.split("/")[0])
    t["conversion"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = O.cg(lambda v: O.spmv(final, rep, v, workers=4), b, tol=1e-300, max_iters=iters)
    per_it = (time.perf_counter() - t0) / max(1, res["iterations"])
    nnz, tnnz = csr.cols.size, (3 * target_n3 - 2) ** 3
    scale = tnnz / nnz
    prep = (t["features"] + t["inference"] + t["conversion"]) * scale
    value = prep + per_it * scale * total_iters
    return {"value": value, "phases": {k: v * scale for k, v in t.items()}, "config": final,
            "per_iteration_s": per_it * scale, "sampled_nnz": int(nnz), "target_nnz": int(tnnz)}


def load_models():
    d = ROOT / "tests" / "golden" / "models"
    return {p.stem: json.loads(p.read_text()) for p in d.glob("*.json")}


def sample(csr: O.OCsr, models, iters: int, total_iters: int, b: np.ndarray) -> dict:
    """One bounded sample of the predict-then-solve pipeline."""
    t = {}
    t0 = time.perf_counter()
    coo = O.csr_to_coo(csr)                      # the user's matrix arrives as COO
    t["to_csr"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    fv = O.features(O.coo_to_csr(coo))
    t["features"] = time.perf_counter() - t0 + t["to_csr"]
    t0 = time.perf_counter()
    final = O.cascade(models, fv)[-1]
    t["inference"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    fmt = final.split("/")[0]
    rep = O.convert(coo, fmt)
    t["conversion"] = time.perf_counter() - t0
    # per-iteration times of Arnoldi steps j = 0..iters-1; step j costs one
    # SpMV plus j+1 MGS dot/axpy pairs, so t_j = a + b*j is fitted and summed
    # over the restart schedule of `total_iters` iterations (restart 30)
    marks = [time.perf_counter()]
    res = O.gmres(lambda v: O.spmv(final, rep, v, workers=4), b, restart=30, tol=1e-300,
                  max_iters=iters, on_iteration=lambda done, j: marks.append(time.perf_counter()))
    # the first step of a cycle also carries the restart (explicit residual,
    # basis allocation), so it is taken as measured and the fit uses j >= 1
    tj = np.diff(np.asarray(marks))
    js = np.arange(tj.size)
    first = float(tj[0])
    slope, icpt = np.polyfit(js[1:], tj[1:], 1) if tj.size >= 3 else (0.0, float(tj[-1]))
    sched = np.arange(total_iters) % 30
    t["solve_extrapolated"] = float(np.sum(np.where(sched == 0, first, icpt + slope * sched)))
    prep = t["features"] + t["inference"] + t["conversion"]
    return {"value": prep + t["solve_extrapolated"], "phases": t, "config": final,
            "per_iteration_s": float(np.mean(icpt + slope * sched)),
            "sampled_iterations": res["iterations"], "fit": [float(icpt), float(slope)]}


def async_full(csr: O.OCsr, b: np.ndarray, models, tol: float = 1e-8, restart: int = 30) -> dict:
    """The reference's async_solve (solver.py:452-493) on the CPU, measured in
    full (nothing extrapolated): the solve starts at once on the reference's
    DEFAULT_CONFIG (COO/LibA, kernels.py:101) while an advisor thread runs
    features -> cascade -> conversion (solver.py:415-449) and publishes one
    update per cascade stage; the solver applies the newest update between
    Arnoldi steps.  b is computed outside the clock (solver.py:470-471)."""
    import threading
    t0 = time.perf_counter()
    coo = O.csr_to_coo(csr)                 # SpmvExecutor.for_matrix(m, DEFAULT_CONFIG)
    state = {"cfg": "COO/LibA", "rep": coo}
    box = {"upd": None}
    lock = threading.Lock()
    cancel = threading.Event()
    swaps = [(1, "COO/LibA", 0.0)]

    def advisor():
        reps = {"COO": coo, "CSR": csr}
        fv = O.features(csr)
        for tok in O.cascade(models, fv):
            if cancel.is_set():
                return
            fmt = tok.split("/")[0]
            t = time.perf_counter()
            if fmt not in reps:
                reps[fmt] = O.convert(coo, fmt)
            with lock:
                box["upd"] = (tok, reps[fmt], time.perf_counter() - t)

    th = threading.Thread(target=advisor, daemon=True)
    th.start()

    def poll(done, j):
        with lock:
            upd, box["upd"] = box["upd"], None
        if upd is not None and upd[0] != state["cfg"]:
            state["cfg"], state["rep"] = upd[0], upd[1]
            swaps.append((done + 1, upd[0], upd[2]))

    res = O.gmres(lambda v: O.spmv(state["cfg"], state["rep"], v, workers=4), b, restart=restart, tol=tol,
                  max_iters=1000, on_iteration=poll)
    cancel.set()
    th.join()
    wall = time.perf_counter() - t0
    return {"value": wall, "iterations": res["iterations"], "converged": res["converged"],
            "final_residual": res["final"], "swaps": swaps}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=2000)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--total-iters", type=int, default=77)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=0)
    ap.add_argument("--laplace27", type=int, default=0,
                    help="config 5 mode: sample grid size (the solve is extrapolated per nnz)")
    ap.add_argument("--target", type=int, default=600, help="config 5: grid size extrapolated to")
    ap.add_argument("--async-full", action="store_true",
                    help="config 2: the reference's async_solve flow, measured in full")
    a = ap.parse_args(argv)
    if a.laplace27:
        r = cg_sample(a.laplace27, a.iters, a.total_iters, a.target, load_models())
        print(json.dumps({"value": r["value"], "unit": "s", "cores": os.cpu_count(),
                          "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"), "kind": "port",
                          "cpu_model": cpu_model(),
                          "sample": (f"reference predict-then-solve with the CG oracle on the 27-point "
                                     f"Laplacian {a.laplace27}^3 (nnz={r['sampled_nnz']:,}), "
                                     f"{a.iters} CG iterations timed; preprocessing and per-iteration "
                                     f"time scaled per nnz to {a.target}^3 (nnz={r['target_nnz']:,}) and "
                                     f"the solve to {a.total_iters} iterations (EXTRAPOLATED)"),
                          "phases": r["phases"], "config": r["config"],
                          "per_iteration_s": r["per_iteration_s"], "sampled_nnz": r["sampled_nnz"]}))
        return 0
    if a.async_full:
        csr = convdiff9_csr(a.nx)
        b = O.spmv_sequential(csr, np.ones(csr.nrows))
        r = async_full(csr, b, load_models())
        r.update({"unit": "s", "cores": os.cpu_count(), "kind": "port", "cpu_model": cpu_model(),
                  "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
                  "sample": (f"reference async_solve flow on conv-diff9 {a.nx}^2 (n={csr.nrows}, "
                             f"nnz={csr.cols.size}), GMRES(30) tol 1e-8 from COO/LibA with the advisor "
                             "thread, measured end to end (not extrapolated)")})
        print(json.dumps(r))
        return 0
    t_gen = time.perf_counter()
    csr = convdiff9_csr(a.nx)
    b = O.spmv_sequential(csr, np.ones(csr.nrows))        # RHS outside the clock (solver.py:355)
    models = load_models()
    t_gen = time.perf_counter() - t_gen
    for _ in range(a.warmup):
        sample(csr, models, a.iters, a.total_iters, b)
    runs = [sample(csr, models, a.iters, a.total_iters, b) for _ in range(a.repeat)]
    vals = sorted(r["value"] for r in runs)
    out = {"value": vals[len(vals) // 2], "values": [r["value"] for r in runs],
           "unit": "s", "cores": os.cpu_count(),
           "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
           "kind": "port", "cpu_model": cpu_model(),
           "sample": (f"reference predict-then-solve on conv-diff9 {a.nx}^2 "
                      f"(n={csr.nrows}, nnz={csr.cols.size}): features+cascade+conversion "
                      f"in full, {runs[0]['sampled_iterations']} GMRES(30) iterations timed "
                      f"and extrapolated to {a.total_iters}"),
           "phases": runs[len(runs) // 2]["phases"], "config": runs[0]["config"],
           "per_iteration_s": runs[len(runs) // 2]["per_iteration_s"],
           "setup_seconds": t_gen}
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
