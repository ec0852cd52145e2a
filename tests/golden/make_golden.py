"""Generate the golden fixtures from the REAL reference implementation.

Run in the build container (the only place ``/root/reference`` exists):

    OPENBLAS_NUM_THREADS=1 SPMVTUNE_WORKERS=4 python tests/golden/make_golden.py

It imports ``spmvtune`` from ``/root/reference/pkg/src`` and the reference's
own test helpers (``tests/helpers.py``: random_coo, poisson2d, banded,
random_feature_array), runs the reference code on a fixed set of matrices
and writes:

  tests/golden/cases/<name>.npz   containers, conversions, features, 13 SpMVs
  tests/golden/models/*.json      the reference's shipped cascade models
  tests/golden/cascade.json       per-model labels/scores on 1000 feature rows
                                  each (stands in for the missing
                                  heldout_predictions.json)
  tests/golden/solves.json        GMRES reports (iterations, history, solution)
  tests/golden/index.json         case list + environment fingerprint

Nothing under tests/ reads /root/reference at run time; the fixtures travel.
"""
from __future__ import annotations

import json
import os
import shutil
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("SPMVTUNE_WORKERS", "4")

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import spmvtune as S  # noqa: E402  (the reference)
import helpers as H   # noqa: E402  (the reference's test helpers)

HERE = Path(__file__).resolve().parent
CASES = HERE / "cases"
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
from paper_2411_10143_b200 import generators as G  # noqa: E402  (inputs only)


def coo_of(n, m, ptr, cols, vals):
    rows = np.repeat(np.arange(n), np.diff(ptr))
    return S.CooMatrix(n, m, rows, cols, vals)


def long_rows_case():
    """Rows long enough to exercise numpy's recursive pairwise split (>128)."""
    rng = np.random.default_rng(77)
    nrows, ncols = 40, 5000
    lens = rng.integers(0, 40, size=nrows)
    lens[[3, 11, 12, 30]] = [129, 300, 1031, 4099]
    rows, cols = [], []
    for i, L in enumerate(lens):
        c = np.sort(rng.choice(ncols, size=int(L), replace=False))
        rows.append(np.full(c.size, i)); cols.append(c)
    rows = np.concatenate(rows); cols = np.concatenate(cols)
    vals = rng.uniform(-1.5, 1.5, size=rows.size)
    return S.CooMatrix.from_triplets(nrows, ncols, rows, cols, vals)


def build_cases():
    cases = {}
    cases["eye3"] = H.coo_from_dense(np.eye(3))
    cases["ones2x3"] = H.coo_from_dense(np.ones((2, 3)))
    cases["gap1x3"] = H.coo_from_dense(np.array([[1.0, 0.0, 1.0]]))
    d = np.zeros((5, 4)); d[0, 3] = 2.0; d[3, 0] = 1.0; d[3, 1] = 4.0
    cases["empty_rows"] = H.coo_from_dense(d)
    cases["zero4x5"] = S.CooMatrix(4, 5, [], [], [])
    cases["poisson10"] = H.poisson2d(10)
    rng = np.random.default_rng(2024)
    for k in range(12):
        cases[f"random{k:02d}"] = H.random_coo(rng, max_n=256, max_density=0.25,
                                               square=(k % 3 == 0))
    cases["banded"] = H.banded(700, [-33, -5, -1, 0, 1, 2, 17, 40],
                               np.random.default_rng(5), diagonal_boost=8.0)
    cases["convdiff24"] = coo_of(*G.convdiff9(24))
    cases["powerlaw3000"] = coo_of(*G.powerlaw_spd(3000, seed=3))
    cases["laplace27_6"] = coo_of(*G.laplace27(6))
    cases["long_rows"] = long_rows_case()
    n = S.DIA_OFFSET_CAP + 10
    cases["dia_overcap"] = S.CooMatrix(n, n, np.zeros(n, dtype=np.int64), np.arange(n),
                                       np.linspace(0.5, 1.5, n))
    return cases


def dump_case(name, coo):
    out = {"nrows": coo.nrows, "ncols": coo.ncols,
           "coo_rows": coo.rows, "coo_cols": coo.cols, "coo_vals": coo.values}
    csr = S.convert(coo, S.FormatTag.CSR)
    out["csr_ptr"] = csr.row_ptr
    ell = S.convert(coo, S.FormatTag.ELL)
    out["ell_width"] = ell.width
    out["ell_cols"] = np.ascontiguousarray(ell.col_idx.T)   # stored (width, nrows)
    out["ell_vals"] = np.ascontiguousarray(ell.values.T)
    try:
        dia = S.convert(coo, S.FormatTag.DIA)
        out["dia_ok"] = 1
        out["dia_offsets"] = dia.offsets
        out["dia_data"] = dia.data
    except S.FormatInapplicableError:
        out["dia_ok"] = 0
    hyb = S.convert(coo, S.FormatTag.HYB)
    out["hyb_width"] = hyb.split_width
    out["hyb_ell_cols"] = np.ascontiguousarray(hyb.ell_part.col_idx.T)
    out["hyb_ell_vals"] = np.ascontiguousarray(hyb.ell_part.values.T)
    out["hyb_spill_rows"] = hyb.coo_part.rows
    out["hyb_spill_cols"] = hyb.coo_part.cols
    out["hyb_spill_vals"] = hyb.coo_part.values
    fv = S.extract_features(csr)
    out["features"] = fv.to_array()
    x = np.random.default_rng(0).uniform(0.5, 1.5, size=coo.ncols)   # bench.py:76-78
    out["x"] = x
    out["y_reference"] = S.spmv_reference(csr, x)
    tokens = []
    for cfg in S.enumerate_configs():
        tok = cfg.token()
        if tok == "COO/LibB":
            continue  # nondeterministic by design (kernels.py:156-164)
        try:
            rep = S.convert(coo, cfg.format)
        except S.FormatInapplicableError:
            continue
        workers_list = (1, 3, 4, 7, 64) if cfg.library is S.Library.LIB_C else (4,)
        for w in workers_list:
            key = f"y|{tok}|{w}"
            out[key] = S.execute_spmv(cfg, rep, x, workers=w)
            tokens.append(key)
    np.savez_compressed(CASES / f"{name}.npz", **out)
    return {"name": name, "nrows": coo.nrows, "ncols": coo.ncols, "nnz": coo.nnz,
            "spmv_keys": tokens, "features": fv.to_array().tolist()}


def dump_cascade(index):
    models_dir = REF / "tests" / "fixtures" / "models"
    dst = HERE / "models"
    dst.mkdir(exist_ok=True)
    for p in sorted(models_dir.glob("*.json")):
        shutil.copyfile(p, dst / p.name)
    models = S.CascadeModelSet.load_dir(models_dir)
    named = {"FORMAT": models.format_model, "COO-LIB": models.coo_lib_model,
             "CSR-LIB": models.csr_lib_model, "ELL-LIB": models.ell_lib_model,
             "CSR-TPV": models.csr_tpv_model}
    rng = np.random.default_rng(4242)
    rows = [H.random_feature_array(rng).tolist() for _ in range(1000)]
    rows += [c["features"] for c in index]
    doc = {"feature_names": list(S.FEATURE_NAMES), "models": {}, "cascade": []}
    for name, model in named.items():
        labels, scores = [], []
        for r in rows:
            lab, sc = model.predict(np.asarray(r))
            labels.append(lab); scores.append(sc.tolist())
        doc["models"][name] = {"rows": rows, "labels": labels, "scores": scores}
    for r in rows:
        decisions = []
        final = S.cascade_predict(models, np.asarray(r), decisions.append)
        doc["cascade"].append({"row": r, "final": final.token(),
                               "decisions": [d.implied_config().token() for d in decisions],
                               "stages": [d.stage.value for d in decisions]})
    (HERE / "cascade.json").write_text(json.dumps(doc))


def dump_solves():
    out = {}

    def run(name, coo, params):
        csr = S.convert(coo, S.FormatTag.CSR)
        b = S.spmv_reference(csr, np.ones(coo.ncols)) if params.rhs == "ones" else None
        rep = S.gmres_solve(coo, b, params,
                            executor=S.SpmvExecutor.for_matrix(
                                coo, S.SpmvConfig(S.FormatTag.CSR, S.Library.LIB_B)))
        out[name] = {"matrix": name.split("@")[0], "restart": params.restart_m,
                     "tol": params.tol, "max_iters": params.max_iters, "rhs": params.rhs,
                     "seed": params.seed,
                     "converged": rep.converged, "iterations": rep.iterations,
                     "history": rep.residual_history, "final": rep.final_residual,
                     "solution": rep.solution.tolist()}

    P = S.GmresParams
    run("poisson10@m30", H.poisson2d(10), P(restart_m=30, tol=1e-8, max_iters=1000))
    run("poisson10@m5", H.poisson2d(10), P(restart_m=5, tol=1e-8, max_iters=2000))
    run("poisson10@forced50", H.poisson2d(10), P(restart_m=30, tol=1e-300, max_iters=50))
    run("convdiff24@m30", coo_of(*G.convdiff9(24)), P(restart_m=30, tol=1e-8))
    run("convdiff24@m10", coo_of(*G.convdiff9(24)), P(restart_m=10, tol=1e-8))
    run("banded@m30", H.banded(700, [-33, -5, -1, 0, 1, 2, 17, 40],
                                np.random.default_rng(5), diagonal_boost=8.0),
        P(restart_m=30, tol=1e-8))
    run("powerlaw3000@random", coo_of(*G.powerlaw_spd(3000, seed=3)),
        P(restart_m=30, tol=1e-8, rhs="random", seed=0))
    (HERE / "solves.json").write_text(json.dumps(out))


def main():
    CASES.mkdir(parents=True, exist_ok=True)
    index = [dump_case(name, coo) for name, coo in build_cases().items()]
    dump_cascade(index)
    dump_solves()
    env = {"numpy": np.__version__, "python": sys.version.split()[0],
           "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
           "SPMVTUNE_WORKERS": os.environ.get("SPMVTUNE_WORKERS"),
           "reference": str(REF / "src" / "spmvtune")}
    (HERE / "index.json").write_text(json.dumps({"env": env, "cases": index}, indent=1))
    print("wrote", len(index), "cases")


if __name__ == "__main__":
    main()
