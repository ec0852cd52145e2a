"""Row-partitioned solver logic with world_size 2 on CPU (gloo).

The distributed driver (paper_2411_10143_b200/distributed.py) is run with
numpy/gloo doubles of its two interfaces: `ops` computes local products with
the CPU oracle, `comm` is torch.distributed over gloo.  What is tested is the
product's partitioning, halo plan, exchange sequencing, all-reduce placement
and solver control flow — against the single-process oracle solve.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2411_10143_b200 import generators as G
from paper_2411_10143_b200.distributed import (HaloPlan, dist_cg, dist_gmres, local_block,
                                                partition_rows, DistOperator)
from paper_2411_10143_b200.features import features_from_aggregates
from paper_2411_10143_b200.solver import GmresParams
from paper_2411_10143_b200.kernels import SpmvConfig


class NumpyOps:
    """Local-kernel test double (numpy + oracle)."""

    def __init__(self, n):
        self.n = n

    def vec(self, n=None):
        return np.zeros(self.n if n is None else n)

    def scalars(self, k):
        return np.zeros(k)

    def view(self, v, off, cnt):
        return v[off:off + cnt]

    def upload(self, v, a):
        v[:] = a

    def fetch(self, v):
        return v.copy()

    def read(self, sc, count):
        return sc[:count].copy()

    def copy(self, dst, src):
        dst[:] = src

    def dot(self, x, y, sc, i):
        sc[i] = float(np.dot(x, y))

    def axpy_dot(self, sc_a, ia, sign, x, y, z, sc_out, io):
        y += sign * sc_a[ia] * x
        if sc_out is not None:
            sc_out[io] = float(np.dot(z if z is not None else y, y))

    def axpby(self, a, x, b, y):
        y[:] = a * x + b * y

    def cg_rupdate(self, sc, icur, ipq, out, ialpha, q, r):
        pq = sc[ipq]
        ok = pq != 0.0 and np.isfinite(pq)
        sc[ialpha] = sc[icur] / pq if ok else 0.0
        if ok:
            r -= sc[ialpha] * q
            sc[out] = float(np.dot(r, r))
        else:
            sc[out] = sc[icur]

    def cg_xp(self, sc, ialpha, inew, iold, r, p, x):
        x += sc[ialpha] * p
        p[:] = r + (sc[inew] / sc[iold]) * p

    GS_DOT, GS_UPDATE, GS_FINISH, GS_AXPY = 0, 1, 2, 3

    def basis(self, rows):
        return _NpBasis(np.zeros((rows, self.n)))

    def gs(self, mode, V, k, sc_h, ih, w, dst, sc_out, io, sc_div=None, idiv=0):
        B = V.a[:k]
        if mode == self.GS_DOT:
            sc_out[io:io + k] = B @ w
            return
        h = sc_h[ih:ih + k]
        t = w + h @ B if mode == self.GS_AXPY else w - h @ B
        if mode == self.GS_FINISH:
            t = t / sc_div[idiv]
        dst[:] = t
        if mode == self.GS_UPDATE:
            sc_out[io:io + k] = B @ dst
            sc_out[io + k] = float(dst @ dst)

    def gs_hn(self, sc, ih2, k, inrm, ihn):
        r = sc[inrm] - float(np.sum(sc[ih2:ih2 + k] ** 2))
        sc[ihn] = np.sqrt(r) if r > 0 else 0.0

    def maxpy(self, V, k, coef, x):
        x += coef[:k] @ V.a[:k]

    def read_async(self, sc, count):
        return sc[:count].copy()

    def read_wait(self, token):
        return token

    def scale(self, x, s):
        x *= s

    def prepare(self, block, cfg):
        if block.nloc == 0:
            return None
        csr = O.OCsr(block.nloc, block.window, block.row_ptr, block.cols, block.values)
        return O.convert(csr, cfg.format.value) if cfg.format.value != "CSR" else csr

    def prepare_rows(self, block, cfg, a, b):
        s, e = int(block.row_ptr[a]), int(block.row_ptr[b])
        csr = O.OCsr(b - a, block.window, block.row_ptr[a:b + 1] - s, block.cols[s:e],
                     block.values[s:e])
        return O.convert(csr, cfg.format.value) if cfg.format.value != "CSR" else csr

    def spmv(self, mat, cfg, window, dst):
        if mat is None:
            return
        dst[:] = O.spmv(cfg.token(), mat, window, workers=4)


class _NpBasis:
    def __init__(self, a):
        self.a = a

    def row(self, i):
        return self.a[i]


class GlooComm:
    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def allreduce(self, sc, first, count):
        t = self.torch.from_numpy(sc[first:first + count])
        self.dist.all_reduce(t)

    def allgather_obj(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def exchange(self, sends, recvs):
        self.exchange_finish(self.exchange_start(sends, recvs))

    def exchange_start(self, sends, recvs):
        # the halo is written only at finish, so an interior SpMV run in
        # between sees the previous step's halo: a row misclassified as
        # interior changes the result
        reqs = [self.dist.isend(self.torch.from_numpy(np.ascontiguousarray(v)), p) for p, v in sends]
        bufs = [(v, self.torch.zeros(v.size, dtype=self.torch.float64)) for _, v in recvs]
        reqs += [self.dist.irecv(t, p) for (p, _), (_, t) in zip(recvs, bufs)]
        return reqs, bufs

    def exchange_finish(self, token):
        reqs, bufs = token
        for r in reqs:
            r.wait()
        for v, t in bufs:
            v[:] = t.numpy()


class NumpyPeerComm(GlooComm):
    """Test double of PeerComm's halo push: the x/p pass publishes the rows
    each neighbour needs (addresses = fake per-rank window bases + the same
    offset arithmetic DistOperator.setup_push uses), and they land in the
    window only at wait_halo — after the interior rows ran, as a late
    NVLink push would — so a misplaced segment or a missing wait changes
    the solve."""

    def alloc(self, n):
        return np.zeros(n)

    def share_buffer(self, buf):
        self._win, self._pending = buf, []
        return [q << 40 for q in range(self.world)]

    def xp_push(self, n, sc, ialpha, inew, iold, r, p, x, segs):
        x += sc[ialpha] * p
        p[:] = r + (sc[inew] / sc[iold]) * p
        msgs = [(peer, dst, p[lo:lo + cnt].copy()) for lo, cnt, dst, peer in segs]
        for got in self.allgather_obj(msgs):
            self._pending += [(dst, d) for peer, dst, d in got if peer == self.rank]

    def wait_halo(self, peers):
        for dst, d in self._pending:
            off = (dst - (self.rank << 40)) // 8
            self._win[off:off + d.size] = d
        self._pending = []

    def check(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, _, ptr, cols, vals = case["gen"]()
        bounds = partition_rows(ptr, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        blk = local_block(ptr, cols, vals, r0, r1, n)
        ops, comm = NumpyOps(blk.nloc), (NumpyPeerComm() if case.get("peer") else GlooComm())
        A = DistOperator(blk, bounds, comm, ops, SpmvConfig.from_token(case["cfg"]))
        csr = O.OCsr(n, n, ptr, cols, vals)
        b = O.spmv_sequential(csr, np.ones(n))
        params = GmresParams(restart_m=case.get("restart", 30), tol=1e-8, max_iters=3000)
        res = (dist_cg if case["method"] == "cg" else dist_gmres)(A, b[r0:r1], params)
        # global features from per-rank aggregates (a rank without rows adds
        # nothing and stays out of the min)
        if blk.nloc:
            lc = O.OCsr(blk.nloc, blk.window, blk.row_ptr, blk.cols, blk.values)
            a = O.feature_aggregates(lc)
            mine = (a["sum_r"], a["sum_r2"], a["max_r"], a["min_r"], a["span"], a["runs"])
        else:
            mine = (0, 0, 0, None, 0, 0)
        parts = comm.allgather_obj(mine + (blk.offsets.tolist(),))
        agg = (sum(p[0] for p in parts), sum(p[1] for p in parts), max(p[2] for p in parts),
               min(p[3] for p in parts if p[3] is not None), sum(p[4] for p in parts),
               sum(p[5] for p in parts), len(set().union(*[set(p[6]) for p in parts])))
        fv = features_from_aggregates(n, n, int(ptr[-1]), agg).to_array().tolist()
        q.put((rank, r0, r1, res["iterations"], res["converged"], res["final"], res["x"], fv,
               HaloPlan.build(bounds, comm.allgather_obj((blk.cmin, blk.cmax)), rank), A.split,
               res.get("allreduces"), res.get("arnoldi_steps"), res.get("halo_push")))
    finally:
        dist.destroy_process_group()


CASES = {
    "cg-poisson-dia": {"gen": lambda: G.poisson2d(24), "method": "cg", "cfg": "DIA/LibA"},
    "gmres-restart40-csr": {"gen": lambda: G.convdiff9(22), "method": "gmres", "cfg": "CSR/LibB",
                            "restart": 40},
    "cg-empty-rank-world4": {"gen": lambda: G.poisson2d(2), "method": "cg", "cfg": "CSR/LibB",
                             "world": 6},
    "cg-dia-peer-push": {"gen": lambda: G.poisson2d(24), "method": "cg", "cfg": "DIA/LibA", "peer": True},
    "cg-csr-peer-push-world3": {"gen": lambda: G.poisson2d(30), "method": "cg", "cfg": "CSR/LibB", "world": 3,
                                "peer": True},
    "cg-laplace27-peer-push-world4": {"gen": lambda: G.laplace27(12), "method": "cg", "cfg": "DIA/LibA",
                                      "world": 4, "peer": True},
    "cg-peer-push-empty-ranks": {"gen": lambda: G.stencil_csr((7,), [(-1,), (0,), (1,)], [-1.0, 2.5, -1.0]),
                                 "method": "cg", "cfg": "DIA/LibA", "world": 9, "peer": True},
    "gmres-empty-rank-world5": {"gen": lambda: G.convdiff9(2), "method": "gmres", "cfg": "CSR/LibB",
                                "world": 5},
    "gmres-convdiff-csr": {"gen": lambda: G.convdiff9(20), "method": "gmres", "cfg": "CSR/LibB"},
    "gmres-powerlaw-ell": {"gen": lambda: G.powerlaw_spd(600, seed=5), "method": "gmres",
                           "cfg": "ELL/LibA"},
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_row_partitioned_solve_world2(name):
    import multiprocessing as mp
    case = CASES[name]
    world = case.get("world", 2)
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, _, ptr, cols, vals = case["gen"]()
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    mv = lambda v: O.spmv("CSR/LibB", csr, v)          # noqa: E731
    ref = (O.cg(mv, b, tol=1e-8, max_iters=3000) if case["method"] == "cg"
           else O.gmres(mv, b, restart=case.get("restart", 30), tol=1e-8, max_iters=3000))
    x = np.concatenate([o[6] for o in outs])
    assert outs[0][1] == 0 and outs[-1][2] == n
    assert all(outs[k][2] == outs[k + 1][1] for k in range(world - 1))
    if "empty" in name:
        assert any(o[2] == o[1] for o in outs)          # some rank really owns no rows
    if case["method"] == "gmres":                       # CGS2: two all-reduces per Arnoldi step
        for o in outs:
            assert o[10] <= 2 * o[11] + 2 + 3 * 4, (o[10], o[11])
    if case.get("peer"):                                # the halo travelled by push, not exchange
        assert all(o[12] for o in outs)
    for o in outs:
        assert o[3] == outs[0][3]                       # ranks agree
        assert o[4] and o[5] <= 1e-8
    assert abs(outs[0][3] - ref["iterations"]) <= 1
    assert np.linalg.norm(x - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    assert outs[0][7] == O.features(csr)                # exact global features
    if name in ("cg-poisson-dia", "gmres-convdiff-csr", "gmres-restart40-csr"):   # interior overlaps the halo
        assert all(o[9] is not None for o in outs)
    for o in outs:                                      # halo symmetric
        plan = o[8]
        for peer, lo, hi in plan.recvs:
            assert (o[0], lo, hi) in [(q_, l_, h_) for q_, l_, h_ in outs[peer][8].sends]


def test_partition_balances_nnz():
    n, _, ptr, cols, vals = G.powerlaw_spd(5000, seed=1)
    for world in (1, 2, 3, 8):
        b = partition_rows(ptr, world)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        loads = np.diff(ptr[b])
        assert loads.max() <= ptr[-1] / world + np.diff(ptr).max() + 1


def test_stencil_halo_is_neighbour_planes():
    n, _, ptr, cols, vals = G.laplace27(12)
    bounds = partition_rows(ptr, 4)
    blocks = [local_block(ptr, cols, vals, int(bounds[r]), int(bounds[r + 1]), n) for r in range(4)]
    windows = [(b.cmin, b.cmax) for b in blocks]
    for r in range(4):
        plan = HaloPlan.build(bounds, windows, r)
        peers = sorted(p for p, _, _ in plan.recvs)
        assert peers == [p for p in (r - 1, r + 1) if 0 <= p < 4]
        assert plan.bytes_per_exchange() <= 8 * 2 * (12 * 12 + 12 + 1)


def _stencil27():
    offs, w = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dz, dy, dx))
                w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
    return offs, w


@pytest.mark.parametrize("dims,world", [((7, 5, 4), 3), ((9, 6), 4), ((4, 3, 3), 4), ((5, 5, 5), 1)])
def test_stencil_slab_windows_cover_brute_force(dims, world):
    """z-slab partition of a device-generated stencil: whole planes per rank,
    and the column window / global diagonal set equal what the rows of the
    host CSR hold (the device block generator relies on both)."""
    from paper_2411_10143_b200.distributed import stencil_block_window, stencil_partition
    if len(dims) == 3:
        offs, w = _stencil27()
    else:
        offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
        w = [8.5 if o == (0, 0) else -1.0 for o in offs]
    n, _, ptr, cols, _ = G.stencil_csr(dims, offs, w)
    bounds = stencil_partition(dims, world)
    plane = int(np.prod(dims[1:]))
    assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) >= 0)
    assert np.all(bounds % plane == 0)
    for r in range(world):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        if r0 == r1:
            continue
        cmin, cmax, present = stencil_block_window(dims, offs, r0, r1)
        c = cols[ptr[r0]:ptr[r1]]
        rows = np.repeat(np.arange(r0, r1), np.diff(ptr[r0:r1 + 1]))
        # the window covers every column the rows touch (it may be a few
        # entries wider than the tight range: the generator bounds it by the
        # stencil reach) and the diagonal set is exact
        assert cmin <= min(int(c.min()), r0) and cmax >= max(int(c.max()), r1 - 1)
        reach = int(np.abs(present).max())
        assert cmin >= max(0, r0 - reach) and cmax <= min(n - 1, r1 - 1 + reach)
        assert present.tolist() == np.unique(c - rows).tolist()


@pytest.mark.parametrize("gen,world", [(lambda: G.laplace27(9), 3), (lambda: G.convdiff9(17), 4),
                                       (lambda: G.powerlaw_spd(800, seed=2), 2),
                                       (lambda: G.poisson2d(12), 1)])
def test_interior_rows_read_only_own_columns(gen, world):
    """interior_rows: every row of the run reads only this rank's own rows
    (host blocks exactly; device stencil blocks from the diagonal reach),
    and the run is the longest such run for host blocks."""
    from paper_2411_10143_b200.distributed import LocalBlock, interior_rows
    n, _, ptr, cols, vals = gen()
    bounds = partition_rows(ptr, world)
    for r in range(world):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        blk = local_block(ptr, cols, vals, r0, r1, n)
        rows = np.repeat(np.arange(blk.nloc), np.diff(blk.row_ptr))
        g = blk.cols + blk.cmin
        bad = np.zeros(blk.nloc, dtype=bool)
        np.logical_or.at(bad, rows, (g < r0) | (g >= r1))
        for b in (blk, LocalBlock(blk.r0, blk.r1, blk.cmin, blk.cmax, None, None, None, n,
                                  blk.offsets)):
            sp = interior_rows(b, min_fraction=0.0)
            if world == 1:
                assert sp is None
                continue
            if sp is None:                  # the reach-based rule may be conservative
                assert bad.all() or b.row_ptr is None
                continue
            ia, ib = sp
            assert 0 <= ia < ib <= blk.nloc and not bad[ia:ib].any()
            if b.row_ptr is not None:
                runs = np.diff(np.flatnonzero(np.concatenate(([True], bad, [True]))))
                assert ib - ia == runs.max() - 1
