"""BASELINE-scale fixtures, generated from the REAL reference in this container.

    OPENBLAS_NUM_THREADS=1 SPMVTUNE_WORKERS=4 python tests/golden/make_scale_fixtures.py [config ...]

The matrices of BASELINE.json configs 1-3 are far too large to commit, so
this script stores SCALARS and HASHES only (tests/golden/scale.json):

* the sha256 of the CSR arrays (row_ptr int64, col_idx int64, values f64) of
  the generated matrix, so the GPU test proves it multiplies the same matrix;
* per SpMV configuration, the sha256 of the reference's y = execute_spmv(cfg,
  convert(A, fmt), x, workers=4) for x = rng(0).uniform(0.5, 1.5, n) (the
  reference's time_config input, bench.py:81-106) — the bit-exact target —
  plus |y|_2 and the sequential spmv_reference hash for the atomic COO/LibB;
* the reference's 15 features and cascade decision (shipped models);
* solves: config 2 GMRES(30) with the reference's own gmres_solve on DIA;
  configs 1 and 3 with the CG oracle (oracle/cpu_oracle.cg — the reference
  has no CG) whose matvec is the REFERENCE's execute_spmv in
  the cascade's chosen kernel.  Iterations, final residual, first history
  entries.

Nothing under tests/ reads /root/reference at run time; scale.json travels.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("SPMVTUNE_WORKERS", "4")

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

import spmvtune as S  # noqa: E402  (the reference)

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
import oracle as O  # noqa: E402  (CG restatement only)
from paper_2411_10143_b200 import generators as G  # noqa: E402  (inputs only)

OUT = HERE / "scale.json"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def matrix(name: str):
    if name == "config1":
        return G.poisson2d(1024)
    if name == "config2":
        return G.convdiff9(2000)
    if name == "config3":
        return G.powerlaw_spd(8_000_000, seed=0)
    if name == "config5_120":
        return G.laplace27(120)     # config 5's matrix family at 120^3 (600^3 has 5.8 B nnz)
    if name == "config2_8M":
        return G.convdiff9(2830)    # config 2's family above the on-chip Arnoldi capacity (4.85 M rows)
    if name in ("convdiff_362", "convdiff_512"):
        return G.convdiff9(int(name.split("_")[1]))   # config 2's family where the Arnoldi kernel runs on 32 / 64 CTAs
    raise KeyError(name)


def spmv_hashes(csr, x, skip=()) -> dict:
    out = {}
    reps = {S.FormatTag.CSR: csr}
    for cfg in S.enumerate_configs():
        tok = cfg.token()
        if cfg.format.value in skip:
            continue
        if cfg.format not in reps:
            t = time.perf_counter()
            try:
                reps[cfg.format] = S.convert(csr, cfg.format)
            except S.FormatInapplicableError as exc:
                reps[cfg.format] = exc
            print(f"  convert {cfg.format.value}: {time.perf_counter() - t:.1f}s", flush=True)
        rep = reps[cfg.format]
        if isinstance(rep, Exception):
            out[tok] = {"inapplicable": str(rep)}
            continue
        t = time.perf_counter()
        y = S.execute_spmv(cfg, rep, x, workers=4)
        out[tok] = {"sha256": sha(y), "norm": float(np.linalg.norm(y))}
        print(f"  {tok}: {time.perf_counter() - t:.1f}s", flush=True)
    return out


def cg_oracle(csr, tok, b, tol=1e-8, max_iters=20000) -> dict:
    cfg = S.SpmvConfig.from_token(tok) if hasattr(S.SpmvConfig, "from_token") else None
    if cfg is None:
        parts = tok.split("/")
        cfg = S.SpmvConfig(S.FormatTag(parts[0]), S.Library(parts[1]),
                           int(parts[2]) if len(parts) > 2 else None)
    rep = csr if cfg.format is S.FormatTag.CSR else S.convert(csr, cfg.format)
    t = time.perf_counter()
    r = O.cg(lambda v: S.execute_spmv(cfg, rep, v, workers=4), b, tol=tol, max_iters=max_iters)
    return {"matvec": tok, "iterations": int(r["iterations"]), "converged": bool(r["converged"]),
            "final_residual": float(r["final"]), "history_head": [float(v) for v in r["history"][:5]],
            "seconds": time.perf_counter() - t}


def build_gmres_only(name: str) -> dict:
    """config2_8M / convdiff_362 / convdiff_512: the matrix hash and the
    reference's GMRES(30) on DIA only (the parity targets of the partially
    resident and the reduced-grid Arnoldi kernels)."""
    t0 = time.perf_counter()
    n, m, ptr, cols, vals = matrix(name)
    doc = {"n": int(n), "nnz": int(cols.size),
           "csr_sha256": sha(np.asarray(ptr, np.int64), np.asarray(cols, np.int64), np.asarray(vals, np.float64))}
    csr = S.CsrMatrix(n, m, ptr, cols, vals)
    params = S.GmresParams(restart_m=30, tol=1e-8, max_iters=1000)
    dia = S.convert(csr, S.FormatTag.DIA)
    t = time.perf_counter()
    rep = S.gmres_solve(dia, None, params,
                        executor=S.SpmvExecutor(S.SpmvConfig(S.FormatTag.DIA, S.Library.LIB_A), dia))
    doc["gmres30"] = {"iterations": rep.iterations, "converged": rep.converged,
                      "final_residual": float(rep.final_residual),
                      "history_head": [float(v) for v in rep.residual_history[:5]],
                      "seconds": time.perf_counter() - t, "matvec": "DIA/LibA"}
    doc["seconds"] = time.perf_counter() - t0
    return doc


def build(name: str, models) -> dict:
    if name in ("config2_8M", "convdiff_362", "convdiff_512"):
        return build_gmres_only(name)
    t0 = time.perf_counter()
    n, m, ptr, cols, vals = matrix(name)
    print(f"{name}: n={n} nnz={cols.size} generated in {time.perf_counter() - t0:.1f}s", flush=True)
    doc = {"n": int(n), "nnz": int(cols.size),
           "csr_sha256": sha(np.asarray(ptr, np.int64), np.asarray(cols, np.int64), np.asarray(vals, np.float64))}
    csr = S.CsrMatrix(n, m, ptr, cols, vals)
    x = np.random.default_rng(0).uniform(0.5, 1.5, size=m)
    doc["spmv_reference_sha256"] = sha(S.spmv_reference(csr, x))
    doc["spmv"] = spmv_hashes(csr, x, skip=("ELL", "DIA") if name == "config3" else
                              ("COO", "ELL", "HYB") if name == "config5_120" else ())
    fv = S.extract_features(csr)
    doc["features"] = [float(v) for v in fv.to_array()]
    stages = []
    final = S.cascade_predict(models, fv, lambda d: stages.append(d.implied_config().token()))
    doc["cascade"] = {"stages": stages, "final": final.token()}
    if name == "config2":
        params = S.GmresParams(restart_m=30, tol=1e-8, max_iters=1000)
        dia = S.convert(csr, S.FormatTag.DIA)
        t = time.perf_counter()
        rep = S.gmres_solve(dia, None, params,
                            executor=S.SpmvExecutor(S.SpmvConfig(S.FormatTag.DIA, S.Library.LIB_A), dia))
        doc["gmres30"] = {"iterations": rep.iterations, "converged": rep.converged,
                          "final_residual": float(rep.final_residual),
                          "history_head": [float(v) for v in rep.residual_history[:5]],
                          "seconds": time.perf_counter() - t, "matvec": "DIA/LibA"}
    elif name == "config1":
        b = S.spmv_reference(csr, np.ones(n))
        doc["cg"] = cg_oracle(csr, "DIA/LibA", b)
    elif name == "config3":
        b = np.random.default_rng(0).standard_normal(n)      # rhs="random", seed 0 (solver.py:190-191)
        doc["cg"] = cg_oracle(csr, "CSR/LibB", b)
    elif name == "config5_120":
        # the bench's predict-then-solve CG (b = A*1, the cascade's kernel)
        b = S.spmv_reference(csr, np.ones(n))
        doc["cg"] = cg_oracle(csr, final.token(), b)
        dia = S.convert(csr, S.FormatTag.DIA)
        r = O.cg(lambda v: S.execute_spmv(S.SpmvConfig(S.FormatTag.DIA, S.Library.LIB_A), dia, v, workers=4), b,
                 tol=1e-8, max_iters=20000)
        doc["cg"]["x_norm"] = float(np.linalg.norm(r["x"]))
        doc["cg"]["x_head"] = [float(v) for v in r["x"][:4]]
    doc["seconds"] = time.perf_counter() - t0
    return doc


def main(argv):
    names = argv or ["config1", "config2", "config3"]
    models = S.CascadeModelSet.load_dir(HERE / "models")
    doc = json.loads(OUT.read_text()) if OUT.exists() else {}
    doc["environment"] = {"numpy": np.__version__, "OPENBLAS_NUM_THREADS": os.environ["OPENBLAS_NUM_THREADS"],
                          "SPMVTUNE_WORKERS": os.environ["SPMVTUNE_WORKERS"],
                          "x": "np.random.default_rng(0).uniform(0.5, 1.5, n)"}
    for name in names:
        doc[name] = build(name, models)
        OUT.write_text(json.dumps(doc, indent=1, sort_keys=True))
        print(f"{name} done in {doc[name]['seconds']:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
