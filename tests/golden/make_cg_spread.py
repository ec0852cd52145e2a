"""How far the reference's own CG iteration count moves when only the
summation order of its inner products changes (config 3: power-law SPD,
8 M rows, b random seed 0, tol 1e-8, CSR/LibB matvec — bit-exact to the
reference kernel).  The reference computes inner products with BLAS ddot
(np.dot), whose order depends on the CPU's OpenBLAS kernel and thread
count; every variant below is an equally valid fp64 inner
product:

  blas1     np.dot, OPENBLAS_NUM_THREADS=1 (the scale.json fixture)
  pairwise  numpy's pairwise sum of the rounded products
  exact     math.fsum of the rounded products (correctly rounded sum)
  blocked   two-level sum of 1024-element blocks (a GPU-style tree)

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_cg_spread.py

writes config3.cg_spread into tests/golden/scale.json.  The GPU test then
holds the CUDA CG to [min - 1, max + 1] of this spread (an ill-conditioned
CG run of ~300 iterations is not reproducible to +-1 across dot orders —
not by the reference itself either)."""
from __future__ import annotations

import json
import math
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
import oracle as O  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402

DOTS = {
    "blas1": lambda a, b: float(np.dot(a, b)),
    "pairwise": lambda a, b: float(np.sum(a * b)),
    "exact": lambda a, b: math.fsum(a * b),
    "blocked": lambda a, b: float(np.sum(np.add.reduceat(a * b, np.arange(0, a.size, 1024)))),
}
STATE = {}


def run(name):
    csr, b = STATE["csr"], STATE["b"]
    t = time.perf_counter()
    r = O.cg(lambda v: O.spmv("CSR/LibB", csr, v), b, tol=1e-8, max_iters=20000, dot=DOTS[name])
    return name, {"iterations": int(r["iterations"]), "converged": bool(r["converged"]),
                  "final_residual": float(r["final"]), "seconds": time.perf_counter() - t}


def main():
    n, m, ptr, cols, vals = G.powerlaw_spd(8_000_000, seed=0)
    STATE["csr"] = O.OCsr(n, m, ptr, cols, vals)
    STATE["b"] = np.random.default_rng(0).standard_normal(n)
    with mp.get_context("fork").Pool(len(DOTS)) as pool:
        res = dict(pool.map(run, list(DOTS)))
    its = [v["iterations"] for v in res.values()]
    out = HERE / "scale.json"
    doc = json.loads(out.read_text())
    doc["config3"]["cg_spread"] = {"variants": res, "min": min(its), "max": max(its)}
    out.write_text(json.dumps(doc, indent=1, sort_keys=True))
    print(json.dumps(doc["config3"]["cg_spread"]))


if __name__ == "__main__":
    main()
