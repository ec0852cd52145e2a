"""Parity at BASELINE.json sizes (configs 1-3) against fixtures the REAL
reference produced in the build container (tests/golden/make_scale_fixtures.py
-> tests/golden/scale.json: hashes of the reference's SpMV outputs, its
features and cascade decision, its GMRES(30) report; CG reports of the
oracle whose matvec is the reference's own kernel).

Size-dependent code paths only these sizes reach:
  * config 2 (4 M rows): k_mgs_tma's shared-memory chunks of w (slices above
    12,288 elements), every Arnoldi fallback forced through SPMVTUNE_MGS;
  * config 3 (8 M rows, 112 M nnz): power-law row kernels with long rows,
    the HYB spill, the device-built power-law generator;
  * int64 row pointers (nnz >= 2^31 only at config 5) forced on the golden
    cases with SPMVTUNE_FORCE_PTR64=1.
"""
import hashlib
import json
import os
import subprocess
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
MODELS = HERE / "golden" / "models"


@lru_cache(maxsize=None)
def fixtures():
    return json.loads((HERE / "golden" / "scale.json").read_text())


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def stencil_offsets(ndim, center, other):
    import itertools
    offs, w = [], []
    for o in itertools.product((-1, 0, 1), repeat=ndim):
        offs.append(o)
        w.append(center if not any(o) else other(o))
    return offs, w


@lru_cache(maxsize=None)
def matrix(name):
    if name == "config1":
        return P.CsrMatrix.stencil((1024, 1024), [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)],
                                   [4.0, -1.0, -1.0, -1.0, -1.0])
    if name == "config2":
        offs, w = stencil_offsets(2, 8.5, lambda o: -1.0 - 0.25 * (o[1] + o[0]))
        return P.CsrMatrix.stencil((2000, 2000), offs, w)
    if name == "config3":
        return G.powerlaw_spd_device(8_000_000, seed=0)
    if name == "config5_120":       # config 5's 27-point Laplacian family at 120^3
        offs, w = stencil_offsets(3, 26.0, lambda o: -1.0)
        return P.CsrMatrix.stencil((120, 120, 120), offs, w)
    raise KeyError(name)


CONFIGS = ["config1", "config2", "config3", "config5_120"]


@pytest.mark.parametrize("name", CONFIGS)
def test_generated_matrix_is_the_fixture_matrix(name):
    """The device generators build exactly the arrays the reference
    multiplied (config 3: the device radix-sort generator == the numpy one)."""
    f = fixtures()[name]
    A = matrix(name)
    assert (A.nrows, A.nnz) == (f["n"], f["nnz"])
    assert sha(A.row_ptr, A.col_idx, A.values) == f["csr_sha256"]


@pytest.mark.parametrize("name", CONFIGS)
def test_every_spmv_configuration_bit_exact_at_scale(name):
    f = fixtures()[name]
    A = matrix(name)
    x = np.random.default_rng(0).uniform(0.5, 1.5, size=A.ncols)
    yref = P.spmv_reference(A, x)
    assert sha(yref) == f["spmv_reference_sha256"]
    reps = {}
    checked = 0
    for cfg in P.enumerate_configs():
        want = f["spmv"].get(cfg.token())
        if want is None or "inapplicable" in want:
            continue
        if cfg.format not in reps:
            reps[cfg.format] = A if cfg.format is P.FormatTag.CSR else P.convert(A, cfg.format)
        y = P.execute_spmv(cfg, reps[cfg.format], x, workers=4)
        if cfg.token() == "COO/LibB":   # the reference's scatter order is not deterministic either
            assert np.linalg.norm(y - yref) <= 1e-12 * np.linalg.norm(yref)
        else:
            assert sha(y) == want["sha256"], cfg.token()
        checked += 1
    assert checked == sum(1 for v in f["spmv"].values() if "inapplicable" not in v)
    assert checked >= (8 if name == "config5_120" else 10 if name == "config3" else 13)


@pytest.mark.parametrize("name", CONFIGS)
def test_features_and_cascade_at_scale(name):
    f = fixtures()[name]
    A = matrix(name)
    fv = P.extract_features(A)
    assert fv.to_array().tolist() == f["features"]
    stages = []
    final = P.cascade_predict(P.CascadeModelSet.load_dir(MODELS), fv,
                              lambda d: stages.append(d.implied_config().token()))
    assert final.token() == f["cascade"]["final"]
    assert stages == f["cascade"]["stages"]


def test_config2_gmres30_matches_reference_report():
    """GMRES(30) at 4 M rows: the TMA/TMEM Arnoldi kernel with w chunks in
    shared memory (slices of 27K elements).  Reference: 77 iterations."""
    g = fixtures()["config2"]["gmres30"]
    A = matrix("config2")
    params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000)
    for rep in (P.gmres_solve(A, None, params, initial_config=P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)),
                P.async_solve(A, None, params, P.CascadeModelSet.load_dir(MODELS),
                              initial_config=P.GPU_DEFAULT_CONFIG)):
        assert rep.converged == g["converged"]
        assert abs(rep.iterations - g["iterations"]) <= 1
        assert rep.final_residual <= 1e-8
        assert np.allclose(rep.residual_history[:5], g["history_head"], rtol=1e-9, atol=0)


_MGS_SCRIPT = r"""
import json, sys, itertools
sys.path.insert(0, {root!r})
import paper_2411_10143_b200 as P
offs, w = [], []
for o in itertools.product((-1, 0, 1), repeat=2):
    offs.append(o); w.append(8.5 if not any(o) else -1.0 - 0.25 * (o[1] + o[0]))
A = P.CsrMatrix.stencil((2000, 2000), offs, w)
r = P.gmres_solve(A, None, P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000),
                  initial_config=P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A))
print(json.dumps({{"iterations": r.iterations, "converged": r.converged, "final": r.final_residual}}))
"""


@pytest.mark.parametrize("mode", ["resident", "tmem", "stream"])
def test_config2_every_arnoldi_fallback(mode):
    """SPMVTUNE_MGS forces the SM-resident (w in shared memory), TMEM-staged
    and streaming (one launch per MGS pass) Arnoldi kernels at config-2 size."""
    g = fixtures()["config2"]["gmres30"]
    env = dict(os.environ, SPMVTUNE_MGS=mode)
    out = subprocess.run([sys.executable, "-c", _MGS_SCRIPT.format(root=str(ROOT))], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["converged"] and abs(r["iterations"] - g["iterations"]) <= 1 and r["final"] <= 1e-8


_MGS_GATE_SCRIPT = r"""
import json, sys, itertools
sys.path.insert(0, {root!r})
import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import _lib
offs, w = [], []
for o in itertools.product((-1, 0, 1), repeat=2):
    offs.append(o); w.append(8.5 if not any(o) else -1.0 - 0.25 * (o[1] + o[0]))
A = P.CsrMatrix.stencil(({nx}, {nx}), offs, w)
params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000)
cfg = P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)
P.gmres_solve(A, None, P.GmresParams(restart_m=30, tol=1e-8, max_iters=3), initial_config=cfg)
l0 = _lib.launch_count()
r = P.gmres_solve(A, None, params, initial_config=cfg)
print(json.dumps({{"iterations": r.iterations, "converged": r.converged, "final": r.final_residual,
                  "launches": _lib.launch_count() - l0}}))
"""


def test_tma_arnoldi_beyond_the_resident_kernels_limit():
    """n = 2180^2 = 4.75 M rows: above the SM-resident kernel's shared-memory
    bound (~4.29 M) but within the TMA kernel's own (148 x 32768 = 4.85 M):
    the TMA/TMEM Arnoldi kernel runs (a few launches per step, not one per MGS
    pass) and lands within 1 iteration of the streaming fallback."""
    res = {}
    for mode in ("default", "stream"):
        env = dict(os.environ)
        env.pop("SPMVTUNE_MGS", None)
        if mode == "stream":
            env["SPMVTUNE_MGS"] = "stream"
        out = subprocess.run([sys.executable, "-c", _MGS_GATE_SCRIPT.format(root=str(ROOT), nx=2180)], env=env,
                             capture_output=True, text=True, timeout=900)
        assert out.returncode == 0, out.stderr[-2000:]
        res[mode] = json.loads(out.stdout.strip().splitlines()[-1])
    a, b = res["default"], res["stream"]
    assert a["converged"] and b["converged"] and a["final"] <= 1e-8 and b["final"] <= 1e-8
    assert abs(a["iterations"] - b["iterations"]) <= 1
    # streaming: one launch per MGS pass (j + 2 per step); TMA: one per step
    assert a["launches"] / a["iterations"] < 6 < b["launches"] / b["iterations"], res


def test_tma_arnoldi_partially_resident_matches_reference():
    """n = 2830^2 = 8.0 M rows: each SM's slice (54 K doubles) exceeds the
    on-chip capacity (32 K), so the TMA kernel runs partially resident (16
    chunks on chip, the rest with w in the V[j+1] row and V_{i-1} streamed):
    one launch per Arnoldi step, within 1 iteration of the reference's
    GMRES(30) (fixture config2_8M, made with the reference's own
    gmres_solve on DIA) and of the streaming fallback."""
    f = fixtures()["config2_8M"]
    res = {}
    for mode in ("default", "stream"):
        env = dict(os.environ)
        env.pop("SPMVTUNE_MGS", None)
        if mode == "stream":
            env["SPMVTUNE_MGS"] = "stream"
        out = subprocess.run([sys.executable, "-c", _MGS_GATE_SCRIPT.format(root=str(ROOT), nx=2830)], env=env,
                             capture_output=True, text=True, timeout=1200)
        assert out.returncode == 0, out.stderr[-2000:]
        res[mode] = json.loads(out.stdout.strip().splitlines()[-1])
    a, b = res["default"], res["stream"]
    assert a["converged"] and b["converged"] and a["final"] <= 1e-8 and b["final"] <= 1e-8
    assert abs(a["iterations"] - f["gmres30"]["iterations"]) <= 1, (a, f["gmres30"])
    assert abs(a["iterations"] - b["iterations"]) <= 1
    assert a["launches"] / a["iterations"] < 6 < b["launches"] / b["iterations"], res


def test_config1_cg_matches_oracle_iterations():
    c = fixtures()["config1"]["cg"]
    A = matrix("config1")
    params = P.GmresParams(tol=1e-8, max_iters=5000)
    for rep in (P.cg_solve(A, None, params, initial_config=P.SpmvConfig.from_token(c["matvec"])),
                P.async_solve(A, None, params, P.CascadeModelSet.load_dir(MODELS), method="cg",
                              initial_config=P.GPU_DEFAULT_CONFIG)):
        assert rep.converged and abs(rep.iterations - c["iterations"]) <= 1
        assert rep.final_residual <= 1e-8


def test_config3_cg_within_the_references_own_spread():
    """Config 3 is ill-conditioned (~300 CG iterations): the iteration count
    moves with the summation order of the inner products alone — the
    reference's np.dot order depends on the CPU's BLAS kernel and thread
    count.  tests/golden/make_cg_spread.py reran the oracle CG (bit-exact
    reference matvec) with four valid fp64 inner-product orders; the CUDA CG
    (device tree reductions) must land within that spread +-1."""
    c = fixtures()["config3"]["cg"]
    spread = fixtures()["config3"].get("cg_spread", {"min": c["iterations"], "max": c["iterations"]})
    lo, hi = spread["min"] - 1, spread["max"] + 1
    A = matrix("config3")
    params = P.GmresParams(tol=1e-8, max_iters=20000, rhs="random", seed=0)
    for rep in (P.cg_solve(A, None, params, initial_config=P.SpmvConfig.from_token(c["matvec"])),
                P.async_solve(A, None, params, P.CascadeModelSet.load_dir(MODELS), method="cg",
                              initial_config=P.GPU_DEFAULT_CONFIG)):
        assert rep.converged and lo <= rep.iterations <= hi, (rep.iterations, spread)
        assert rep.final_residual <= 1e-8
        assert np.allclose(rep.residual_history[:5], c["history_head"], rtol=1e-9, atol=0)


def test_int64_row_pointers_on_the_golden_cases():
    """The int64-row-pointer kernels (used when nnz >= 2^31, i.e. config 5 on
    one GPU) forced on every golden case: the SpMV, conversion and feature
    parity suites re-run bit-exact with SPMVTUNE_FORCE_PTR64=1."""
    env = dict(os.environ, SPMVTUNE_FORCE_PTR64="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                          str(HERE / "test_gpu_spmv.py"), str(HERE / "test_gpu_convert_features.py"),
                          str(HERE / "test_gpu_edge_cases.py")],
                         env=env, capture_output=True, text=True, timeout=1200, cwd=str(ROOT))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " passed" in out.stdout and "failed" not in out.stdout


def test_config5_family_row_partitioned_cg_matches_reference():
    """The bench's path (device-generated slab, exact global features ->
    shipped cascade -> DIA, row-partitioned CG over NCCL at world 1) on
    config 5's matrix family at 120^3 against the reference-driven fixture:
    same kernel choice, iterations within 1, residual <= tol, same x."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2411_10143_b200.distributed import distributed_stencil_solve
    f = fixtures()["config5_120"]
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        offs, w = stencil_offsets(3, 26.0, lambda o: -1.0)
        params = P.GmresParams(tol=1e-8, max_iters=20000)
        res, blk = distributed_stencil_solve("cg", (120, 120, 120), offs, w, params,
                                             models=P.CascadeModelSet.load_dir(MODELS))
        assert sha(np.asarray(blk._dev_csr.row_ptr, np.int64), np.asarray(blk._dev_csr.col_idx, np.int64),
                   blk._dev_csr.values) == f["csr_sha256"]
        assert res["config"] == f["cascade"]["final"]
        assert res["converged"] and res["final"] <= 1e-8
        assert abs(res["iterations"] - f["cg"]["iterations"]) <= 1
        x = res["x"].to_numpy()
        # two CG runs with different dot-product orders, both stopped at
        # relative residual <= 1e-8: x agrees to the solve's own accuracy
        assert abs(np.linalg.norm(x) - f["cg"]["x_norm"]) <= 1e-8 * f["cg"]["x_norm"]
        assert np.allclose(x[:4], f["cg"]["x_head"], rtol=1e-7, atol=0)
        assert np.allclose(res["history"][:5], f["cg"]["history_head"], rtol=1e-9, atol=0)
    finally:
        dist.destroy_process_group()


_GRID_SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G
n, m, ptr, cols, vals = G.convdiff9({nx})
A = P.convert(P.CsrMatrix(n, m, ptr, cols, vals), P.FormatTag.DIA)
r = P.gmres_solve(A, None, P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000),
                  initial_config=P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A))
print(json.dumps({{"iterations": r.iterations, "converged": r.converged, "final": r.final_residual,
                  "head": r.residual_history[:5]}}))
"""


@pytest.mark.parametrize("name,nx", [("convdiff_362", 362), ("convdiff_512", 512)])
def test_reduced_grid_arnoldi_matches_reference(name, nx):
    """131 K / 262 K rows: the TMA Arnoldi kernel runs on 32 / 64 CTAs (one
    per 4096 rows, csrc/krylov.cu mgs_grid) instead of one per SM.  Both
    grids land on the reference's own GMRES(30) run (fixtures made with the
    reference's gmres_solve on DIA): same iteration count within 1, final
    residual and the first residual estimates to 1e-6 relative."""
    f = fixtures()[name]["gmres30"]
    for grid in (None, "148"):
        env = dict(os.environ)
        env.pop("SPMVTUNE_MGS", None)
        env.pop("SPMVTUNE_MGS_GRID", None)
        if grid:
            env["SPMVTUNE_MGS_GRID"] = grid
        out = subprocess.run([sys.executable, "-c", _GRID_SCRIPT.format(root=str(ROOT), nx=nx)], env=env,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        r = json.loads(out.stdout.strip().splitlines()[-1])
        assert r["converged"] and abs(r["iterations"] - f["iterations"]) <= 1, (grid, r, f)
        assert abs(r["final"] - f["final_residual"]) <= 1e-6 * f["final_residual"], (grid, r, f)
        assert np.allclose(r["head"], f["history_head"], rtol=1e-6, atol=0), (grid, r, f)
