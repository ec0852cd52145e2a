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


def _world2_worker(rank, port, method, dims, q, cfg=None, p2p="1"):
    """One of two ranks sharing the single test GPU: CUDA kernels, device
    halo windows and device scalars; collectives staged through gloo
    (HostStagedComm) or, with p2p="1", the peer-memory layer on top of it
    (PeerComm over CUDA IPC between the two processes: mailbox all-reduces,
    halo pushed by the x/p pass)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPMVTUNE_P2P=p2p)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2411_10143_b200.distributed import HostStagedComm, distributed_stencil_solve
        offs, w = _stencil(dims)
        params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=3000)
        models = P.CascadeModelSet.load_dir(os.path.join(os.path.dirname(__file__), "golden", "models"))
        if cfg is None:
            res, blk = distributed_stencil_solve(method, dims, offs, w, params, models=models,
                                                 comm_class=HostStagedComm)
        else:
            res, blk = distributed_stencil_solve(method, dims, offs, w, params,
                                                 initial_config=P.SpmvConfig.from_token(cfg),
                                                 comm_class=HostStagedComm)
        q.put((rank, blk.r0, blk.r1, res["iterations"], res["converged"], res["final"],
               res["x"].to_numpy(), res["config"], blk.cmin, blk.cmax, res["interior_rows"],
               res.get("peer_collectives"), res.get("halo_push")))
    except Exception as exc:          # surface worker failures in the parent
        import traceback
        q.put((rank, "error", repr(exc) + traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


def _stencil(dims):
    if len(dims) == 3:
        offs, w = [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    offs.append((dz, dy, dx))
                    w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
        return offs, w
    offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    return offs, [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]


@pytest.mark.parametrize("method,dims,cfg,p2p", [("cg", (14, 12, 10), None, "1"), ("gmres", (44, 40), None, "1"),
                                                 ("cg", (14, 12, 10), "DIA/LibA", "1"),
                                                 ("cg", (14, 12, 10), "DIA/LibA", "0")])
def test_cuda_path_world2_on_one_gpu(method, dims, cfg, p2p):
    """World size 2 of the CUDA row-partitioned path (two processes on the
    one GPU, gloo-staged collectives): the halo exchange really moves planes
    between ranks, interior rows are multiplied while it is in flight;
    iterations within 1 of the oracle and the assembled x matches it."""
    import multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_world2_worker, args=(r, port, method, dims, q, cfg, p2p)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    errors = [o for o in out if o[1] == "error"]
    assert not errors, errors
    offs, w = _stencil(dims)
    n, _, ptr, cols, vals = G.stencil_csr(dims, offs, w)
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    mv = lambda v: O.spmv("CSR/LibB", csr, v)      # noqa: E731
    ref = O.cg(mv, b, tol=1e-8, max_iters=3000) if method == "cg" else \
        O.gmres(mv, b, restart=30, tol=1e-8, max_iters=3000)
    (_, a0, a1, it0, c0, f0, x0, cfg0, _, cmax0, sp0, pc0, hp0), \
        (_, b0, b1, it1, c1, f1, x1, cfg1, cmin1, _, sp1, pc1, hp1) = out
    # the peer-memory layer ran (CUDA IPC between the two processes) unless disabled
    assert pc0 == pc1 == (p2p == "1")
    if method == "cg":
        assert hp0 == hp1 == (p2p == "1")      # the halo travelled by push in the x/p pass
    assert a0 == 0 and a1 == b0 and b1 == n and cmax0 >= a1 and cmin1 < b0   # real halos both ways
    # the interior rows' SpMV ran before the halo landed (HostStagedComm
    # writes it at exchange_finish), the boundary rows after
    assert sp0 is not None and sp1 is not None
    assert it0 == it1 and c0 and c1 and f0 == f1 and f0 <= 1e-8
    assert abs(it0 - ref["iterations"]) <= 1
    x = np.concatenate([x0, x1])
    assert np.linalg.norm(x - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    if cfg is not None:
        assert cfg0 == cfg1 == cfg
        return
    fv = P.extract_features(P.CsrMatrix(n, n, ptr, cols, vals))
    assert cfg0 == cfg1 == P.cascade_predict(
        P.CascadeModelSet.load_dir(os.path.join(os.path.dirname(__file__), "golden", "models")), fv).token()


@pytest.mark.parametrize("a,b", [(0, 1), (0, 600), (17, 430), (599, 600), (123, 124)])
def test_csr_row_slice_is_exact(a, b):
    """svb_csr_row_slice (the interior/boundary blocks of a rank): the arrays
    equal the host slice with a rebased row pointer, and the row-local SpMV
    configurations give exactly the full SpMV's rows."""
    from paper_2411_10143_b200.formats import CsrMatrix, _new_handle
    from paper_2411_10143_b200 import _lib
    n, _, ptr, cols, vals = G.powerlaw_spd(600, seed=3)
    A = P.CsrMatrix(n, n, ptr, cols, vals)
    dev = _new_handle(_lib.lib().svb_csr_row_slice, A._device().handle, a, b, None)
    S = CsrMatrix._wrap(dev)
    s, e = int(ptr[a]), int(ptr[b])
    assert (S.nrows, S.ncols, S.nnz) == (b - a, n, e - s)
    assert np.array_equal(S.row_ptr, ptr[a:b + 1] - s)
    assert np.array_equal(S.col_idx, cols[s:e]) and np.array_equal(S.values, vals[s:e])
    x = np.random.default_rng(0).uniform(0.5, 1.5, n)
    for tok in ("CSR/LibB", "CSR/LibA/4", "CSR/LibA/32"):
        cfg = P.SpmvConfig.from_token(tok)
        assert np.array_equal(P.execute_spmv(cfg, S, x), P.execute_spmv(cfg, A, x)[a:b])
    with pytest.raises(ValueError):
        _new_handle(_lib.lib().svb_csr_row_slice, A._device().handle, 5, 5, None)
