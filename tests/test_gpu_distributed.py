"""The row-partitioned driver on the GPU with the production CudaOps/NcclComm
(world size 1 on the single test GPU: exercises the device primitives and
the NCCL all-reduce plumbing; the multi-rank exchange logic is covered by
tests/test_distributed.py on gloo)."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G
from paper_2411_10143_b200.distributed import distributed_solve

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("method,gen", [("cg", "poisson"), ("gmres", "convdiff")])
def test_distributed_solve_world1(nccl_world1, method, gen):
    n, _, ptr, cols, vals = G.poisson2d(48) if gen == "poisson" else G.convdiff9(40)
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=3000)
    models = P.CascadeModelSet.load_dir(os.path.join(os.path.dirname(__file__), "golden", "models"))
    res, bounds = distributed_solve(method, ptr, cols, vals, b, params, models=models)
    mv = lambda v: O.spmv("CSR/LibB", csr, v)      # noqa: E731
    ref = O.cg(mv, b, tol=1e-8, max_iters=3000) if method == "cg" else \
        O.gmres(mv, b, restart=30, tol=1e-8, max_iters=3000)
    assert res["converged"] and res["final"] <= 1e-8
    assert abs(res["iterations"] - ref["iterations"]) <= 1
    assert np.linalg.norm(res["x"] - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    # the cascade ran on global features: same config as the single-GPU prediction
    fv = P.extract_features(P.CsrMatrix(n, n, ptr, cols, vals))
    assert res["config"] == P.cascade_predict(models, fv).token()


def test_stencil_rows_generator_matches_global_rows():
    """svb_csr_stencil_rows = rows [r0, r1) of the global generator with the
    columns shifted by the window start (bit-exact)."""
    from paper_2411_10143_b200.distributed import stencil_block, stencil_partition
    offs, w = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dz, dy, dx))
                w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
    dims = (9, 7, 6)
    n, _, ptr, cols, vals = G.stencil_csr(dims, offs, w)
    bounds = stencil_partition(dims, 3)
    for r in range(3):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        blk = stencil_block(dims, offs, w, r0, r1)
        m = blk._dev_csr
        assert m.nrows == r1 - r0 and m.ncols == blk.window
        assert np.array_equal(np.asarray(m.row_ptr), ptr[r0:r1 + 1] - ptr[r0])
        assert np.array_equal(np.asarray(m.col_idx), cols[ptr[r0]:ptr[r1]] - blk.cmin)
        assert np.array_equal(np.asarray(m.values), vals[ptr[r0]:ptr[r1]])


@pytest.mark.parametrize("method,dims", [("cg", (12, 11, 10)), ("gmres", (40, 36))])
def test_distributed_stencil_solve_world1(nccl_world1, method, dims):
    """Device-generated slab + row-partitioned solve (the config-5 path) vs
    the oracle on the same matrix: iterations within 1, residual <= tol."""
    from paper_2411_10143_b200.distributed import distributed_stencil_solve
    if len(dims) == 3:
        offs, w = [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    offs.append((dz, dy, dx))
                    w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
    else:
        offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
        w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
    n, _, ptr, cols, vals = G.stencil_csr(dims, offs, w)
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=3000)
    models = P.CascadeModelSet.load_dir(os.path.join(os.path.dirname(__file__), "golden", "models"))
    t = {}
    res, blk = distributed_stencil_solve(method, dims, offs, w, params, models=models, timings=t)
    mv = lambda v: O.spmv("CSR/LibB", csr, v)      # noqa: E731
    ref = O.cg(mv, b, tol=1e-8, max_iters=3000) if method == "cg" else \
        O.gmres(mv, b, restart=30, tol=1e-8, max_iters=3000)
    assert res["converged"] and res["final"] <= 1e-8
    assert abs(res["iterations"] - ref["iterations"]) <= 1
    x = res["x"].to_numpy() if hasattr(res["x"], "to_numpy") else np.asarray(res["x"])
    assert np.linalg.norm(x - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    fv = P.extract_features(P.CsrMatrix(n, n, ptr, cols, vals))
    assert res["config"] == P.cascade_predict(models, fv).token()
    assert t["total_s"] > 0
