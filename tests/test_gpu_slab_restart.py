"""GPU tests for the per-rank host-slab entry point (distributed_solve_slab,
svb_csr_create_slab / svb_csr_export / svb_diag_offsets), ranks that own no
rows, restart lengths beyond 63 — each against the CPU oracle."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G
from paper_2411_10143_b200.distributed import device_diag_offsets, local_block, slab_block

pytestmark = pytest.mark.gpu
MODELS = os.path.join(os.path.dirname(__file__), "golden", "models")


def _slab(ptr, cols, vals, r0, r1):
    s, e = int(ptr[r0]), int(ptr[r1])
    return ptr[r0:r1 + 1] - s, cols[s:e], vals[s:e]


@pytest.mark.parametrize("gen,r0,r1,idx", [("powerlaw", 700, 2100, np.int64), ("powerlaw", 0, 3000, np.int32),
                                           ("convdiff", 1000, 2000, np.int32), ("convdiff", 2599, 3600, np.int64)])
def test_slab_block_equals_the_host_block(gen, r0, r1, idx):
    """Window, window-relative columns and global diagonal offsets computed
    on the device from a host slab equal the host slicing (local_block)."""
    n, _, ptr, cols, vals = G.powerlaw_spd(3000, seed=5) if gen == "powerlaw" else G.convdiff9(60)
    p, c, v = _slab(ptr, cols, vals, r0, r1)
    blk = slab_block(r0, r1, n, p, c.astype(idx), v)
    ref = local_block(ptr, cols, vals, r0, r1, n)
    assert (blk.cmin, blk.cmax, blk.nloc) == (ref.cmin, ref.cmax, ref.nloc)
    A = blk._dev_csr
    assert np.array_equal(A.row_ptr, ref.row_ptr) and np.array_equal(A.col_idx, ref.cols)
    assert np.array_equal(A.values, ref.values)
    assert np.array_equal(blk.offsets, ref.offsets)


def test_diag_offsets_and_export_round_trip():
    n, _, ptr, cols, vals = G.banded(5000, [-900, -2, 0, 1, 33, 4000], seed=1, diagonal_boost=1.0)
    A = P.CsrMatrix(n, n, ptr, cols, vals)
    rows = np.repeat(np.arange(n), np.diff(ptr))
    assert np.array_equal(device_diag_offsets(A, 0), np.unique(cols - rows))
    assert np.array_equal(device_diag_offsets(A, 17), np.unique(cols - rows) + 17)
    from paper_2411_10143_b200 import _lib
    hp = np.empty(n + 1, np.int64)
    hc = np.empty(A.nnz, np.int32)
    hv = np.empty(A.nnz)
    _lib.check(_lib.lib().svb_csr_export(A._device().handle, 5, hp.ctypes.data, hc.ctypes.data,
                                         hv.ctypes.data, None))
    assert np.array_equal(hp, ptr) and np.array_equal(hc, cols + 5) and np.array_equal(hv, vals)


def test_slab_validation_matches_csrmatrix_messages():
    n, _, ptr, cols, vals = G.poisson2d(10)
    p, c, v = _slab(ptr, cols, vals, 20, 60)
    cases = []
    bad = p.copy(); bad[5], bad[6] = bad[6], bad[5]
    cases.append(((bad, c, v), "non-decreasing"))
    bad = c.copy(); bad[3] = n
    cases.append(((p, bad, v), "out of range"))
    bad = c.copy(); bad[1], bad[2] = bad[2], bad[1]
    cases.append(((p, bad, v), "strictly increasing"))
    bad = p.copy(); bad[-1] += 1
    cases.append(((bad, c, np.append(v, 1.0)[:v.size]), "endpoints"))
    for (pp, cc, vv), msg in cases:
        with pytest.raises(ValueError, match=msg):
            slab_block(20, 60, n, pp, cc, vv)


@pytest.mark.parametrize("m", [64, 100, 300])
def test_gmres_restart_lengths_beyond_63(m):
    """restart_m >= 64 (the reference accepts any m >= 1): y staged in
    dynamic shared memory, the TMA Arnoldi kernel up to m = 252 and the
    SM-resident kernels beyond."""
    n, _, ptr, cols, vals = G.convdiff9(48)
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    A = P.CsrMatrix(n, n, ptr, cols, vals)
    params = P.GmresParams(restart_m=m, tol=1e-10, max_iters=2000)
    rep = P.gmres_solve(A, b, params, initial_config=P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_B))
    ref = O.gmres(lambda v: O.spmv("CSR/LibB", csr, v), b, restart=m, tol=1e-10, max_iters=2000)
    assert rep.converged and ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= 1
    assert np.linalg.norm(rep.solution - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])


def test_gmres_restart_cap_is_a_value_error():
    n, _, ptr, cols, vals = G.poisson2d(4)
    with pytest.raises(ValueError):
        P.gmres_solve(P.CsrMatrix(n, n, ptr, cols, vals), None, P.GmresParams(restart_m=30000))


# ---------------------------------------------------------------------------
# multi-rank on the one test GPU (gloo-staged collectives)
# ---------------------------------------------------------------------------
def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stencil3(dims):
    offs, w = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dz, dy, dx))
                w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
    return offs, w


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_10143_b200.distributed import (HostStagedComm, distributed_solve_slab,
                                                        distributed_stencil_solve, partition_rows)
        params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=3000)
        models = P.CascadeModelSet.load_dir(MODELS)
        if case == "empty_rank":
            dims = (2, 9, 11)            # 2 planes over 3 ranks: one rank owns nothing
            offs, w = _stencil3(dims)
            res, blk = distributed_stencil_solve("cg", dims, offs, w, params, models=models,
                                                 comm_class=HostStagedComm)
            x = res["x"].to_numpy()
            q.put((rank, blk.r0, blk.r1, res["iterations"], res["converged"], res["final"], x, res["config"]))
        else:
            method = "cg" if case == "slab_cg" else "gmres"
            n, _, ptr, cols, vals = G.powerlaw_spd(4000, seed=9) if method == "cg" else G.convdiff9(50)
            b = O.spmv_sequential(O.OCsr(n, n, ptr, cols, vals), np.ones(n))
            bounds = partition_rows(ptr, world)
            r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
            p, c, v = _slab(ptr, cols, vals, r0, r1)
            res = distributed_solve_slab(method, r0, r1, n, p, c.astype(np.int32 if rank else np.int64), v,
                                         b[r0:r1], params, models=models, comm_class=HostStagedComm)
            q.put((rank, r0, r1, res["iterations"], res["converged"], res["final"], res["x"], res["config"]))
    except Exception as exc:
        import traceback
        q.put((rank, "error", repr(exc) + traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    errors = [o for o in out if o[1] == "error"]
    assert not errors, errors
    return out


def test_rank_without_rows_idles_through_the_solve():
    out = _run(3, "empty_rank")
    dims = (2, 9, 11)
    offs, w = _stencil3(dims)
    n, _, ptr, cols, vals = G.stencil_csr(dims, offs, w)
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    ref = O.cg(lambda v: O.spmv("CSR/LibB", csr, v), b, tol=1e-8, max_iters=3000)
    assert sorted(o[2] - o[1] for o in out).count(0) == 1          # one rank really is empty
    its = {o[3] for o in out}
    assert len(its) == 1 and abs(its.pop() - ref["iterations"]) <= 1
    assert all(o[4] and o[5] <= 1e-8 for o in out)
    x = np.concatenate([o[6] for o in out])
    assert np.linalg.norm(x - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    fv = P.extract_features(P.CsrMatrix(n, n, ptr, cols, vals))
    assert {o[7] for o in out} == {P.cascade_predict(P.CascadeModelSet.load_dir(MODELS), fv).token()}


@pytest.mark.parametrize("case", ["slab_cg", "slab_gmres"])
def test_distributed_solve_slab_world2(case):
    """Each rank passes only its own host slab (int64 columns on rank 0,
    int32 on rank 1): window, halo plan and global features come from the
    device; iterations within 1 of the oracle, x matches, cascade = the
    single-matrix prediction."""
    out = _run(2, case)
    n, _, ptr, cols, vals = G.powerlaw_spd(4000, seed=9) if case == "slab_cg" else G.convdiff9(50)
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    mv = lambda v: O.spmv("CSR/LibB", csr, v)      # noqa: E731
    ref = O.cg(mv, b, tol=1e-8, max_iters=3000) if case == "slab_cg" else \
        O.gmres(mv, b, restart=30, tol=1e-8, max_iters=3000)
    assert out[0][1] == 0 and out[0][2] == out[1][1] and out[1][2] == n
    assert out[0][3] == out[1][3] and abs(out[0][3] - ref["iterations"]) <= 1
    assert all(o[4] and o[5] <= 1e-8 for o in out)
    x = np.concatenate([out[0][6], out[1][6]])
    assert np.linalg.norm(x - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    fv = P.extract_features(P.CsrMatrix(n, n, ptr, cols, vals))
    assert out[0][7] == out[1][7] == P.cascade_predict(P.CascadeModelSet.load_dir(MODELS), fv).token()
