"""Row-partitioned CG / GMRES across GPUs.

One process per GPU (torchrun), NCCL over NVLink/NVSwitch for the exchange:

* rows are split into contiguous blocks balanced by nnz (``partition_rows``);
* every rank stores its block as a local CSR whose columns index a *window*
  ``[cmin, cmax]`` of the global vector; the window is filled before each
  SpMV by a halo exchange (``HaloPlan``: each peer sends exactly the slice of
  its own rows that falls in my window — the neighbouring planes for a
  stencil, wider ranges for irregular matrices);
* dot products are computed locally into DEVICE scalars and summed in place
  with an all-reduce, so scalars never leave the GPU inside a step; the host
  reads one small block per iteration (GMRES: the Hessenberg column and
  ||w||^2, after which the Givens update runs on the host exactly as the
  reference's _gmres_core does; CG: p.Ap and r.r);
* the cascade runs on GLOBAL features: the seven integer aggregates are
  all-reduced (sum / max / min) and the diagonal count is the union of the
  ranks' diagonal-offset sets, so the predicted configuration equals the
  single-GPU prediction bit for bit.

The driver is written against two small interfaces — ``ops`` (local vector
kernels) and ``comm`` (collectives) — so the same control flow runs with
``CudaOps``/``NcclComm`` in production and with numpy/gloo doubles in the
CPU test suite (tests/test_distributed.py).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib, device
from .errors import SolverNumericalError, StagnationError
from .features import FeatureVector, device_aggregates, features_from_aggregates
from .formats import CsrMatrix, FormatTag, convert
from .kernels import Library, SpmvConfig, default_workers, launch

__all__ = ["partition_rows", "LocalBlock", "local_block", "HaloPlan", "DistOperator", "CudaOps",
           "NcclComm", "HostStagedComm", "interior_rows", "dist_gmres", "dist_cg", "global_features", "distributed_solve",
           "stencil_partition", "stencil_block_window", "stencil_block", "distributed_stencil_solve",
           "slab_block", "device_diag_offsets", "distributed_solve_slab", "PeerComm", "peer_comm_or_base"]


# ---------------------------------------------------------------------------
# partition and halo plan (pure host logic)
# ---------------------------------------------------------------------------
def partition_rows(row_ptr: np.ndarray, world: int) -> np.ndarray:
    """Contiguous row bounds [0 = b0 <= ... <= b_world = n] balancing nnz."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n, nnz = row_ptr.size - 1, int(row_ptr[-1])
    if nnz == 0:
        return np.linspace(0, n, world + 1).astype(np.int64)
    targets = (np.arange(world + 1, dtype=np.float64) * nnz / world)
    b = np.searchsorted(row_ptr, targets, side="left").astype(np.int64)
    b[0], b[-1] = 0, n
    return np.maximum.accumulate(np.minimum(b, n))


@dataclass
class LocalBlock:
    """Rank-local CSR rows [r0, r1) with columns relative to the window."""

    r0: int
    r1: int
    cmin: int
    cmax: int
    row_ptr: np.ndarray
    cols: np.ndarray          # window-relative
    values: np.ndarray
    ncols_global: int
    offsets: np.ndarray       # distinct global diagonal offsets (col - row) of the block

    @property
    def nloc(self) -> int:
        return self.r1 - self.r0

    @property
    def window(self) -> int:
        return self.cmax - self.cmin + 1


def local_block(row_ptr, col_idx, values, r0: int, r1: int, ncols: int) -> LocalBlock:
    """Slice rows [r0, r1) of a global host CSR into a windowed local block.
    The window always covers the rank's own rows so the local slice of x
    lives inside it."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    s, e = int(row_ptr[r0]), int(row_ptr[r1])
    cols = np.asarray(col_idx[s:e], dtype=np.int64)
    cmin = min(int(cols.min()) if cols.size else r0, r0)
    cmax = max(int(cols.max()) if cols.size else r1 - 1, r1 - 1)
    lp = row_ptr[r0:r1 + 1] - s
    rows = np.repeat(np.arange(r0, r1, dtype=np.int64), np.diff(lp))
    offs = np.unique(cols - rows)
    return LocalBlock(r0, r1, cmin, cmax, lp, cols - cmin, np.asarray(values[s:e], np.float64),
                      int(ncols), offs)


# ---------------------------------------------------------------------------
# stencil matrices generated per rank on the device (configs 2 and 5 at
# scale: a 600^3 slab never exists on the host)
# ---------------------------------------------------------------------------
def _stencil_lin(dims, offsets) -> np.ndarray:
    dims = [int(d) for d in dims]
    strides = np.cumprod([1] + dims[::-1][:-1])[::-1]
    return np.asarray(offsets, dtype=np.int64).reshape(-1, len(dims)) @ strides


def stencil_partition(dims, world: int) -> np.ndarray:
    """Row bounds of `world` slabs of whole leading-axis planes (z-slabs for
    a 3-D grid), as even as the plane count allows."""
    planes = int(dims[0])
    plane = int(np.prod([int(d) for d in dims[1:]], dtype=np.int64))
    cuts = np.linspace(0, planes, world + 1).round().astype(np.int64)
    return cuts * plane


def stencil_block_window(dims, offsets, r0: int, r1: int):
    """(cmin, cmax, global diagonal offsets present) of the slab rows
    [r0, r1), which must be whole leading-axis planes."""
    dims = [int(d) for d in dims]
    offs = np.asarray(offsets, dtype=np.int64).reshape(-1, len(dims))
    plane = int(np.prod(dims[1:], dtype=np.int64))
    z0, z1 = r0 // plane, r1 // plane
    lin = _stencil_lin(dims, offsets)
    present = []
    for o, l in zip(offs, lin):
        ok = max(z0, -o[0]) < min(z1, dims[0] - o[0])
        ok = ok and all(abs(int(o[a])) < dims[a] for a in range(1, len(dims)))
        if ok:
            present.append(int(l))
    n = int(np.prod(dims, dtype=np.int64))
    lo = min(present) if present else 0
    hi = max(present) if present else 0
    cmin = min(max(0, r0 + lo), r0)
    cmax = max(min(n - 1, r1 - 1 + hi), r1 - 1)
    return cmin, cmax, np.unique(np.asarray(present, dtype=np.int64))


def stencil_block(dims, offsets, weights, r0: int, r1: int, stream=None) -> "LocalBlock":
    """Rank-local block of a stencil matrix generated on this rank's GPU
    (svb_csr_stencil_rows); no host copy of the rows is made."""
    import ctypes
    if int(r1) == int(r0):
        return _empty_block(int(r0), int(np.prod([int(d) for d in dims])))
    cmin, cmax, present = stencil_block_window(dims, offsets, r0, r1)
    d = np.ascontiguousarray(dims, dtype=np.int64)
    o = np.ascontiguousarray(offsets, dtype=np.int32).reshape(-1)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    from .formats import _new_handle
    dev = _new_handle(_lib.lib().svb_csr_stencil_rows, int(d.size),
                      d.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(w.size),
                      o.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                      w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(r0), int(r1), int(cmin),
                      int(cmax), stream.handle if stream is not None else None)
    blk = LocalBlock(int(r0), int(r1), int(cmin), int(cmax), None, None, None,
                     int(np.prod(d)), present)
    blk._dev_csr = CsrMatrix._wrap(dev)
    return blk


def slab_block(r0: int, r1: int, ncols: int, row_ptr, col_idx, values, stream=None) -> "LocalBlock":
    """Rank-local block from this rank's own HOST slab: rows [r0, r1) with a
    slab-local row pointer (int64), GLOBAL column indices (int64, the
    reference's dtype, or int32) and float64 values.  The slab is uploaded
    and validated on the device (svb_csr_create_slab: CsrMatrix rules,
    formats.py:113-138), its column window is the hull of its columns and
    own rows, and its global diagonal offsets come from the device bitmap
    (svb_diag_offsets) — the host never scans the slab."""
    nloc = int(r1) - int(r0)
    if nloc == 0:
        return _empty_block(int(r0), int(ncols))
    p = np.ascontiguousarray(row_ptr, dtype=np.int64)
    c = np.asarray(col_idx)
    if c.dtype not in (np.int32, np.int64):
        c = c.astype(np.int64)
    c = np.ascontiguousarray(c)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if p.size != nloc + 1:
        raise ValueError("row_ptr must have nrows+1 entries")
    if c.size != v.size:
        raise ValueError("col_idx and values must have equal length")
    L = _lib.lib()
    win = (ctypes.c_int64 * 2)()
    from .formats import _new_handle
    dev = _new_handle(L.svb_csr_create_slab, nloc, int(ncols), int(v.size), int(r0), p.ctypes.data,
                      c.ctypes.data, 1 if c.dtype == np.int64 else 0, v.ctypes.data,
                      stream.handle if stream is not None else None, win)
    csr = CsrMatrix._wrap(dev)
    cmin, cmax = int(win[0]), int(win[1])
    offs = device_diag_offsets(csr, cmin - int(r0), stream)
    blk = LocalBlock(int(r0), int(r1), cmin, cmax, None, None, None, int(ncols), offs)
    blk._dev_csr = csr
    return blk


def device_diag_offsets(csr: CsrMatrix, shift: int, stream=None) -> np.ndarray:
    """Sorted distinct diagonal offsets (col - row) of a device CSR plus
    ``shift`` (svb_diag_offsets)."""
    L = _lib.lib()
    cnt = ctypes.c_int64()
    h = stream.handle if stream is not None else None
    _lib.check(L.svb_diag_offsets(csr._device().handle, int(shift), None, 0, ctypes.byref(cnt), h))
    out = np.empty(max(1, cnt.value), dtype=np.int64)
    _lib.check(L.svb_diag_offsets(csr._device().handle, int(shift),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), out.size,
                                  ctypes.byref(cnt), h))
    return out[:cnt.value]


def _empty_block(r0: int, ncols: int) -> "LocalBlock":
    """A rank that owns no rows (world > planes, or very heavy rows): it
    joins every collective with zero-length vectors and no matrix."""
    blk = LocalBlock(r0, r0, r0, r0 - 1, None, None, None, int(ncols), np.zeros(0, np.int64))
    blk._dev_csr = None
    return blk


@dataclass
class HaloPlan:
    """Who sends which global range to whom.  ``recvs``/``sends`` hold
    (peer, lo, hi) global index ranges; a rank receives the part of its
    window owned by each peer and sends the part of its rows in each peer's
    window."""

    rank: int
    recvs: list
    sends: list

    @classmethod
    def build(cls, bounds, windows, rank: int) -> "HaloPlan":
        world = len(bounds) - 1
        cmin, cmax = windows[rank]
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        recvs, sends = [], []
        for j in range(world):
            if j == rank:
                continue
            lo, hi = max(cmin, int(bounds[j])), min(cmax + 1, int(bounds[j + 1]))
            if lo < hi:
                recvs.append((j, lo, hi))
            pmin, pmax = windows[j]
            lo, hi = max(pmin, r0), min(pmax + 1, r1)
            if lo < hi:
                sends.append((j, lo, hi))
        return cls(rank, recvs, sends)

    def bytes_per_exchange(self) -> int:
        return 8 * sum(hi - lo for _, lo, hi in self.recvs)


def interior_rows(block: LocalBlock, min_fraction: float = 0.25):
    """(ia, ib): the longest contiguous run of local rows whose columns all
    lie in this rank's own rows, so their SpMV can run while the halo
    exchange is in flight; None when there is no halo or the run is below
    ``min_fraction`` of the rows (irregular matrices: nearly every row reads
    a remote column)."""
    n, own = block.nloc, block.r0 - block.cmin
    if n == 0 or (block.cmin >= block.r0 and block.cmax <= block.r1 - 1):
        return None
    if block.row_ptr is None:
        # device-generated stencil slab: row i reads [i + lo, i + hi] (global
        # diagonal offsets), clipped to the grid
        lo, hi = (int(block.offsets.min()), int(block.offsets.max())) if block.offsets.size else (0, 0)
        ia = min(n, max(0, -lo)) if block.cmin < block.r0 else 0
        ib = max(ia, n - max(0, hi)) if block.cmax > block.r1 - 1 else n
    else:
        ptr = np.asarray(block.row_ptr, dtype=np.int64)
        lens = np.diff(ptr)
        flagged = np.zeros(n, dtype=bool)
        nz = np.flatnonzero(lens)
        if nz.size:
            starts = ptr[nz]
            cmin = np.minimum.reduceat(block.cols, starts)
            cmax = np.maximum.reduceat(block.cols, starts)
            flagged[nz] = (cmin < own) | (cmax >= own + n)
        pos = np.concatenate(([-1], np.flatnonzero(flagged), [n]))
        k = int(np.argmax(np.diff(pos)))
        ia, ib = int(pos[k]) + 1, int(pos[k + 1])
    if ib - ia < max(1, int(min_fraction * n)):
        return None
    return ia, ib


# ---------------------------------------------------------------------------
# device implementations of the two interfaces
# ---------------------------------------------------------------------------
class _DevView:
    """(pointer, count) view of float64 device memory, exportable to NCCL."""

    __slots__ = ("ptr", "n")

    def __init__(self, ptr: int, n: int):
        self.ptr, self.n = int(ptr), int(n)

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.n,), "typestr": "<f8", "data": (self.ptr, False), "version": 3,
                "strides": None}


class _Basis:
    """Krylov basis rows in one allocation (row i at buf.ptr + 8*i*ld), the
    layout the block Gram-Schmidt kernels sweep."""

    def __init__(self, buf, ld: int, rows: int, n: int):
        self.buf, self.ld, self.rows, self.n = buf, int(ld), int(rows), int(n)

    def row(self, i: int) -> "_DevView":
        return _DevView(self.buf.ptr + 8 * i * self.ld, self.n)


class CudaOps:
    """Local vector kernels on this rank's GPU (C ABI svb_vec_*)."""

    def __init__(self, n_loc: int, stream: device.Stream):
        self.n = int(n_loc)
        self.stream = stream
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().svb_vecops_create(self.n, ctypes.byref(h)))
        self.h = h.value
        self.L = _lib.lib()

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            try:
                _lib.load().svb_vecops_destroy(h)
            except Exception:
                pass

    # storage
    def vec(self, n: int | None = None) -> device.DeviceVector:
        v = device.DeviceVector(self.n if n is None else n)
        device.memset(v.ptr, 0, v.nbytes, self.stream)
        return v

    def scalars(self, k: int) -> device.DeviceVector:
        return self.vec(k)

    def view(self, v, offset: int, count: int) -> _DevView:
        return _DevView(v.ptr + 8 * offset, count)

    def upload(self, v, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        device.copy(v.ptr, a.ctypes.data, a.nbytes, self.stream)
        self.stream.sync()

    def fetch(self, v) -> np.ndarray:
        return v.to_numpy(self.stream)

    def read(self, sc, count: int) -> np.ndarray:
        out = np.empty(count)
        device.copy(out.ctypes.data, sc.ptr, 8 * count, self.stream)
        self.stream.sync()
        return out

    def copy(self, dst_view: _DevView, src_view: _DevView):
        device.copy(dst_view.ptr, src_view.ptr, 8 * src_view.n, self.stream)

    # kernels
    def dot(self, x, y, sc, i: int):
        _lib.check(self.L.svb_vec_dot(self.h, x.ptr, y.ptr, sc.ptr + 8 * i, self.stream.handle))

    def axpy_dot(self, sc_a, ia: int, sign: float, x, y, z, sc_out, io: int | None):
        _lib.check(self.L.svb_vec_axpy_dot(self.h, sc_a.ptr + 8 * ia, sign, x.ptr, y.ptr,
                                           z.ptr if z is not None else None,
                                           (sc_out.ptr + 8 * io) if sc_out is not None else None,
                                           self.stream.handle))

    def axpby(self, a: float, x, b: float, y):
        _lib.check(self.L.svb_vec_axpby(self.h, a, x.ptr, b, y.ptr, self.stream.handle))

    def scale(self, x, s: float):
        _lib.check(self.L.svb_vec_scale(self.h, x.ptr, s, self.stream.handle))

    # CGS2 block sweeps (svb_vec_gs) over a contiguous basis
    GS_DOT, GS_UPDATE, GS_FINISH, GS_AXPY = 0, 1, 2, 3

    def basis(self, rows: int) -> "_Basis":
        ld = (self.n + 31) & ~31                  # 256-byte aligned rows
        return _Basis(self.vec(rows * ld if self.n else 0), ld, rows, self.n)

    def gs(self, mode: int, V: "_Basis", k: int, sc_h, ih: int, w, dst, sc_out, io: int,
           sc_div=None, idiv: int = 0):
        h = (sc_h.ptr + 8 * ih) if sc_h is not None else None
        out = (sc_out.ptr + 8 * io) if sc_out is not None else None
        div = (sc_div.ptr + 8 * idiv) if sc_div is not None else None
        _lib.check(self.L.svb_vec_gs(self.h, mode, V.buf.ptr, V.ld, k, h, div, w.ptr,
                                     dst.ptr if dst is not None else None, out, self.stream.handle))

    def gs_hn(self, sc, ih2: int, k: int, inrm: int, ihn: int):
        _lib.check(self.L.svb_vec_gs_hn(sc.ptr + 8 * ih2, k, sc.ptr + 8 * inrm, sc.ptr + 8 * ihn,
                                        self.stream.handle))

    def maxpy(self, V: "_Basis", k: int, coef: np.ndarray, x):
        """x += sum_i coef[i] V_i (host coefficients: the back-substituted y)."""
        c = np.ascontiguousarray(coef[:k], dtype=np.float64)
        if getattr(self, "_coef", None) is None or self._coef.n < c.size:
            self._coef = self.vec(max(64, c.size))
        device.copy(self._coef.ptr, c.ctypes.data, c.nbytes, self.stream)
        self.gs(self.GS_AXPY, V, k, self._coef, 0, x, x, None, 0)
        self.stream.sync()              # the host coefficient buffer is a temporary

    def cg_rupdate(self, sc, icur: int, ipq: int, out: int, ialpha: int, q, r):
        _lib.check(self.L.svb_dcg_rupdate(self.h, sc.ptr, icur, ipq, out, ialpha, q.ptr, r.ptr, self.stream.handle))

    def cg_xp(self, sc, ialpha: int, inew: int, iold: int, r, p, x):
        _lib.check(self.L.svb_dcg_xp(self.h, sc.ptr, ialpha, inew, iold, r.ptr, p.ptr, x.ptr, self.stream.handle))

    def read_async(self, sc, count: int):
        """Copy sc[:count] into pinned host memory behind the work enqueued so
        far; read_wait() returns it.  The stream keeps running meanwhile."""
        if getattr(self, "_pin", None) is None:
            h = ctypes.c_void_p()
            _lib.check(self.L.svb_host_alloc(64 * 8, ctypes.byref(h)))
            self._pin = h.value
        device.copy(self._pin, sc.ptr, 8 * count, self.stream)
        return (self.stream.record(), count)

    def read_wait(self, token) -> np.ndarray:
        ev, count = token
        ev.sync()
        return np.ctypeslib.as_array((ctypes.c_double * count).from_address(self._pin)).copy()

    def spmv(self, mat, cfg: SpmvConfig, window, dst):
        if mat is None:          # a rank without rows
            return
        from .solver import DeviceOptions
        timer = DeviceOptions.current().timer    # bench.py: CUDA events around each launch
        if timer is not None:
            timer.begin("spmv:" + cfg.token(), self.stream.handle)
        launch(cfg, mat, window.ptr, dst.ptr, workers=default_workers(), stream=self.stream)
        if timer is not None:
            timer.end("spmv:" + cfg.token(), self.stream.handle)

    def spmv_dot(self, mat, cfg: SpmvConfig, window, dst, dsrc, sc, slot: int, accumulate: bool):
        """dst = A window and sc[slot] (+)= dsrc . dst, fused in one pass on
        DIA (svb_vec_spmv_dot)."""
        from .kernels import _FMT_CODE, _LIB_CODE
        if mat is None:
            if not accumulate:
                device.memset(sc.ptr + 8 * slot, 0, 8, self.stream)
            return
        from .solver import DeviceOptions
        timer = DeviceOptions.current().timer
        if timer is not None:
            timer.begin("spmv:" + cfg.token(), self.stream.handle)
        _lib.check(self.L.svb_vec_spmv_dot(self.h, mat._device().handle, _FMT_CODE[cfg.format],
                                           _LIB_CODE[cfg.library], cfg.lane_width or 0, default_workers(),
                                           window.ptr, dst.ptr, dsrc.ptr, sc.ptr + 8 * slot,
                                           1 if accumulate else 0, self.stream.handle))
        if timer is not None:
            timer.end("spmv:" + cfg.token(), self.stream.handle)

    def local_csr(self, block: LocalBlock) -> CsrMatrix | None:
        if block.nloc == 0:
            return None
        m = getattr(block, "_dev_csr", None)
        if m is None:
            m = CsrMatrix(block.nloc, block.window, block.row_ptr, block.cols, block.values)
            block._dev_csr = m
        return m

    def prepare(self, block: LocalBlock, cfg: SpmvConfig):
        csr = self.local_csr(block)
        if csr is None:
            return None
        return csr if cfg.format is FormatTag.CSR else convert(csr, cfg.format)

    def prepare_rows(self, block: LocalBlock, cfg: SpmvConfig, a: int, b: int):
        """Rows [a, b) of the local block in cfg's format (svb_csr_row_slice
        of the local CSR, cached, then converted)."""
        cache = block.__dict__.setdefault("_row_slices", {})
        csr = cache.get((a, b))
        if csr is None:
            from .formats import _new_handle
            dev = _new_handle(self.L.svb_csr_row_slice, self.local_csr(block)._device().handle,
                              int(a), int(b), self.stream.handle)
            csr = cache[(a, b)] = CsrMatrix._wrap(dev)
        return csr if cfg.format is FormatTag.CSR else convert(csr, cfg.format)


class NcclComm:
    """torch.distributed (NCCL) collectives ordered on the solver stream."""

    def __init__(self, stream: device.Stream):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.ext = torch.cuda.ExternalStream(stream.handle)

    def _t(self, v):
        return self.torch.as_tensor(v if isinstance(v, _DevView) else _DevView(v.ptr, v.n),
                                    device="cuda")

    def allreduce(self, sc, first: int, count: int):
        with self.torch.cuda.stream(self.ext):
            self.dist.all_reduce(self._t(_DevView(sc.ptr + 8 * first, count)))

    def allreduce_max(self, arr: np.ndarray) -> np.ndarray:
        t = self.torch.as_tensor(arr, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().numpy()

    def allgather_obj(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def exchange(self, sends, recvs):
        self.exchange_finish(self.exchange_start(sends, recvs))

    def exchange_start(self, sends, recvs):
        """Enqueue the halo sends/receives behind the work already on the
        solver stream (NCCL's stream waits for it) without making the solver
        stream wait for them: kernels enqueued next overlap the transfer."""
        ops = [self.dist.P2POp(self.dist.isend, self._t(v), peer) for peer, v in sends]
        ops += [self.dist.P2POp(self.dist.irecv, self._t(v), peer) for peer, v in recvs]
        if not ops:
            return []
        with self.torch.cuda.stream(self.ext):
            return self.dist.batch_isend_irecv(ops)

    def exchange_finish(self, works):
        """The solver stream waits for the exchange (device-side wait)."""
        with self.torch.cuda.stream(self.ext):
            for w in works:
                w.wait()


class HostStagedComm:
    """The same collectives over gloo with device buffers staged through the
    host.  Not a production path: it lets the CUDA implementation (CudaOps,
    device halo windows, device scalars) run with several ranks on ONE GPU
    (NCCL refuses two ranks per device), which is how the test suite covers
    world size > 1 of the CUDA path on a single-GPU box."""

    def __init__(self, stream: device.Stream):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.stream = torch, dist, stream
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def _down(self, ptr: int, n: int) -> np.ndarray:
        a = np.empty(n)
        if n:
            device.copy(a.ctypes.data, ptr, 8 * n, self.stream)
            self.stream.sync()
        return a

    def _up(self, ptr: int, a: np.ndarray):
        if a.size:
            device.copy(ptr, a.ctypes.data, a.nbytes, self.stream)
            self.stream.sync()

    def allreduce(self, sc, first: int, count: int):
        a = self._down(sc.ptr + 8 * first, count)
        t = self.torch.from_numpy(a)
        self.dist.all_reduce(t)
        self._up(sc.ptr + 8 * first, a)

    def allreduce_max(self, arr: np.ndarray) -> np.ndarray:
        t = self.torch.from_numpy(np.asarray(arr, dtype=np.float64).copy())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.numpy()

    def allgather_obj(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def exchange(self, sends, recvs):
        self.exchange_finish(self.exchange_start(sends, recvs))

    def exchange_start(self, sends, recvs):
        reqs = [self.dist.isend(self.torch.from_numpy(self._down(v.ptr, v.n)), p) for p, v in sends]
        bufs = [(v, self.torch.zeros(v.n, dtype=self.torch.float64)) for _, v in recvs]
        reqs += [self.dist.irecv(t, p) for (p, _), (_, t) in zip(recvs, bufs)]
        return reqs, bufs

    def exchange_finish(self, token):
        # the halo lands on the stream AFTER whatever was enqueued between
        # start and finish (the interior SpMV), as with NCCL
        reqs, bufs = token
        for r in reqs:
            r.wait()
        for v, t in bufs:
            self._up(v.ptr, t.numpy())


class _PeerBuffer:
    """A cudaMalloc'd float64 buffer (svb_peer_alloc): CUDA-IPC exportable, so
    other ranks' kernels can store into it (the halo windows)."""

    def __init__(self, n: int):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().svb_peer_alloc(8 * int(n), ctypes.byref(h)))
        self.ptr, self.n, self.nbytes = int(h.value), int(n), 8 * int(n)

    def __del__(self):
        ptr, self.ptr = getattr(self, "ptr", 0), 0
        if ptr:
            try:
                _lib.load().svb_peer_free(ptr)
            except Exception:
                pass


class PeerComm:
    """Collectives done by this package's own kernels over NVLink / NVSwitch
    peer memory (csrc/peer.cu) on top of a base comm (NcclComm, or
    HostStagedComm in the one-GPU tests):

    * ``allreduce`` of up to 64 device doubles through the per-rank
      mailboxes (k_peer_allreduce, one tiny kernel on the solver stream, no
      host involvement; bit-identical totals on every rank);
    * the CG loop's halo: the x/p pass pushes the rows each neighbour needs
      straight into the neighbour's window (svb_dcg_xp_push) and the
      neighbour's boundary SpMV waits on the device for the tag
      (svb_peer_wait_halo) — ``DistOperator.setup_push`` builds the plan;
    * everything else (general halo exchanges, object gathers, max
      all-reduces, all-reduces above 64 doubles) goes to the base comm.

    ``ipc``: exchange CUDA IPC handles (one process per GPU); otherwise the
    ranks share one address space and exchange raw device pointers.  Setup
    is collective and fails on every rank together (``PeerSetupError``), so
    callers can fall back to the base comm without desynchronising."""

    MAXC = 64

    class PeerSetupError(RuntimeError):
        pass

    def __init__(self, base, stream: device.Stream, ipc: bool = True):
        self.base, self.stream, self.ipc = base, stream, bool(ipc)
        self.rank, self.world = base.rank, base.world
        self.L = _lib.lib()
        self.h = None
        self._opened: list[int] = []
        ok, err, mb = True, "", None
        try:
            h = ctypes.c_void_p()
            _lib.check(self.L.svb_peer_create(self.rank, self.world, ctypes.byref(h)))
            self.h = h.value
            mbp = ctypes.c_void_p()
            _lib.check(self.L.svb_peer_mailbox(self.h, ctypes.byref(mbp)))
            mb = int(mbp.value)
        except Exception as exc:   # noqa: BLE001 — reported collectively below
            ok, err = False, f"{type(exc).__name__}: {exc}"
        try:
            ptrs = self._share(mb, ok, err)
        except PeerComm.PeerSetupError:
            for d in self._opened:
                self.L.svb_peer_ipc_close(d)
            if self.h is not None:
                self.L.svb_peer_destroy(self.h)
            self._opened, self.h = [], None
            raise
        for q, ptr in enumerate(ptrs):
            _lib.check(self.L.svb_peer_set_mailbox(self.h, q, ptr))

    # -- collective pointer sharing (every step ends in an all-gather, so a
    # failure on one rank is seen by all of them at the same point)
    def _export(self, ptr: int):
        if not self.ipc:
            return ptr
        buf = (ctypes.c_char * 64)()
        _lib.check(self.L.svb_peer_ipc_handle(ptr, buf))
        return bytes(buf)

    def _share(self, ptr: int | None, ok: bool = True, err: str = "") -> list[int]:
        token = None
        if ok:
            try:
                token = self._export(ptr)
            except Exception as exc:   # noqa: BLE001
                ok, err = False, f"{type(exc).__name__}: {exc}"
        got = self.base.allgather_obj((ok, err, token))
        bad = [e for o, e, _ in got if not o]
        if bad:
            raise PeerComm.PeerSetupError(f"peer setup failed on {len(bad)} rank(s): {bad[0]}")
        out, ok, err = [], True, ""
        for q, (_, _, tok) in enumerate(got):
            if q == self.rank or not self.ipc:
                out.append(ptr if q == self.rank else int(tok))
                continue
            try:
                d = ctypes.c_void_p()
                _lib.check(self.L.svb_peer_ipc_open(ctypes.c_char_p(tok), ctypes.byref(d)))
                self._opened.append(int(d.value))
                out.append(int(d.value))
            except Exception as exc:   # noqa: BLE001
                ok, err = False, f"{type(exc).__name__}: {exc}"
                out.append(0)
        fails = [e for o, e in self.base.allgather_obj((ok, err)) if not o]
        if fails:
            raise PeerComm.PeerSetupError(f"peer mapping failed on {len(fails)} rank(s): {fails[0]}")
        return out

    def alloc(self, n: int) -> _PeerBuffer:
        return _PeerBuffer(n)

    def share_buffer(self, buf) -> list[int]:
        """Every rank's ``buf`` (same call on all ranks) as addressable here."""
        return self._share(int(buf.ptr))

    def check(self):
        e = ctypes.c_int(0)
        _lib.check(self.L.svb_peer_error(self.h, ctypes.byref(e)))
        if e.value:
            raise RuntimeError("peer collective timed out (a rank stopped participating)")

    # -- collectives
    def allreduce(self, sc, first: int, count: int):
        if count > self.MAXC:
            return self.base.allreduce(sc, first, count)
        _lib.check(self.L.svb_peer_allreduce(self.h, sc.ptr + 8 * first, int(count), self.stream.handle))

    def allreduce_max(self, arr):
        return self.base.allreduce_max(arr)

    def allgather_obj(self, obj):
        return self.base.allgather_obj(obj)

    def exchange(self, sends, recvs):
        self.base.exchange(sends, recvs)

    def exchange_start(self, sends, recvs):
        return self.base.exchange_start(sends, recvs)

    def exchange_finish(self, token):
        self.base.exchange_finish(token)

    def wait_halo(self, peers):
        arr = (ctypes.c_int32 * max(1, len(peers)))(*peers)
        _lib.check(self.L.svb_peer_wait_halo(self.h, arr, len(peers), self.stream.handle))

    def xp_push(self, n: int, sc, ialpha: int, inew: int, iold: int, r, p, x, segs):
        k = len(segs)
        lo = (ctypes.c_int64 * 2)(*[sg[0] for sg in segs])
        cnt = (ctypes.c_int64 * 2)(*[sg[1] for sg in segs])
        dst = (ctypes.c_void_p * 2)(*[sg[2] for sg in segs])
        peer = (ctypes.c_int32 * 2)(*[sg[3] for sg in segs])
        _lib.check(self.L.svb_dcg_xp_push(self.h, int(n), sc.ptr, ialpha, inew, iold, r.ptr, p.ptr, x.ptr, k,
                                          lo, cnt, dst, peer, self.stream.handle))

    def close(self):
        """Collective: unmap the peers' buffers after everyone is done."""
        if self.h is None:
            return
        self.stream.sync()
        self.base.allgather_obj(None)
        for d in self._opened:
            self.L.svb_peer_ipc_close(d)
        self._opened = []
        self.base.allgather_obj(None)
        self.L.svb_peer_destroy(self.h)
        self.h = None


def peer_comm_or_base(base, stream: device.Stream, ipc: bool = True):
    """PeerComm over ``base`` unless SPMVTUNE_P2P=0, one rank, or the
    collective setup fails (then the base comm, on every rank)."""
    if os.environ.get("SPMVTUNE_P2P", "1") == "0" or base.world == 1:
        return base
    try:
        return PeerComm(base, stream, ipc=ipc)
    except PeerComm.PeerSetupError as exc:
        import warnings
        warnings.warn(f"peer-memory collectives unavailable, using {type(base).__name__}: {exc}")
        return base


# ---------------------------------------------------------------------------
# distributed operator: halo exchange + local SpMV
# ---------------------------------------------------------------------------
class DistOperator:
    def __init__(self, block: LocalBlock, bounds, comm, ops, cfg: SpmvConfig):
        self.block, self.comm, self.ops, self.cfg = block, comm, ops, cfg
        windows = comm.allgather_obj((block.cmin, block.cmax))
        self.plan = HaloPlan.build(bounds, windows, comm.rank)
        self._windows = windows
        # a window other ranks push into must be peer-mappable
        self.window = comm.alloc(block.window) if hasattr(comm, "alloc") else ops.vec(block.window)
        self.push = None
        self.own = block.r0 - block.cmin
        # no halo: the window is exactly this rank's rows (one rank, or a
        # block-diagonal matrix), so the SpMV reads the source vector itself
        self.no_halo = not self.plan.recvs and block.window == block.nloc
        self._own = None
        # interior / boundary split: the interior rows' SpMV overlaps the
        # halo exchange, the boundary rows follow it
        self.split = None
        if (not self.no_halo and self.plan.recvs and hasattr(ops, "prepare_rows")
                and hasattr(comm, "exchange_start")
                and os.environ.get("SPMVTUNE_HALO_OVERLAP", "1") != "0"):
            self.split = interior_rows(block)
        self._prepare(cfg)

    def _prepare(self, cfg: SpmvConfig):
        if self.split is None:
            self.mat, self.parts = self.ops.prepare(self.block, cfg), None
            return
        ia, ib = self.split
        rng = [(ia, ib)] + [(a, b) for a, b in ((0, ia), (ib, self.block.nloc)) if b > a]
        self.mat = None
        self.parts = [(a, b - a, self.ops.prepare_rows(self.block, cfg, a, b)) for a, b in rng]

    def swap(self, cfg: SpmvConfig):
        self.cfg = cfg
        self._prepare(cfg)

    def setup_push(self) -> bool:
        """Collective: map every rank's window and build this rank's halo-push
        segments (local rows [lo, lo+cnt) -> peer window address) for
        PeerComm's x/p pass.  False on every rank unless all can push (<= 2
        neighbours each way, the vector kept in the window)."""
        comm, b = self.comm, self.block
        if not hasattr(comm, "share_buffer"):
            return False
        try:
            ptrs = comm.share_buffer(self.window)
        except PeerComm.PeerSetupError:          # raised on every rank together
            return False
        segs = [(lo - b.r0, hi - lo, ptrs[p] + 8 * (lo - self._windows[p][0]), p)
                for p, lo, hi in self.plan.sends if hi > lo]
        peers = [p for p, lo, hi in self.plan.recvs if hi > lo]
        mine = len(segs) <= 2 and len(peers) <= 2
        if not all(comm.allgather_obj(mine)):
            return False
        self.push = (segs, peers)
        return True

    def apply_dot_pushed(self, src, dst, sc, slot: int):
        """apply_dot when the halo was pushed into this rank's window by the
        neighbours' last x/p pass: the interior rows run at once, the stream
        then waits on the device for the neighbours' tags, then the boundary
        rows.  ``src`` must be the window's own slice (CG's p)."""
        if self.no_halo:                   # nothing to receive: the SpMV reads src itself
            self.apply_dot(src, dst, sc, slot)
            return
        ops = self.ops
        _, peers = self.push
        fused = hasattr(ops, "spmv_dot")

        def part(mat, d, sv, acc):
            if fused:
                ops.spmv_dot(mat, self.cfg, self.window, d, sv, sc, slot, acc)
            else:
                ops.spmv(mat, self.cfg, self.window, d)
        if self.parts is None:
            self.comm.wait_halo(peers)
            part(self.mat, dst, src, False)
        else:
            for k, (a, cnt, mat) in enumerate(self.parts):
                if k == 1:
                    self.comm.wait_halo(peers)
                part(mat, ops.view(dst, a, cnt), ops.view(src, a, cnt), k > 0)
            if len(self.parts) == 1:
                self.comm.wait_halo(peers)
        if not fused:
            ops.dot(src, dst, sc, slot)

    def own_view(self):
        """This rank's slice of the window buffer: a vector kept there (CG's
        p) needs no copy before the halo exchange."""
        if self._own is None:
            self._own = self.ops.view(self.window, self.own, self.block.nloc)
        return self._own

    def apply_dot(self, src, dst, sc, slot: int):
        """dst = A_local * x and sc[slot] = src . dst over the local rows
        (CG's q = A p with p.q): fused into the SpMV pass when ``ops`` can
        (one launch per row part, the parts' dots accumulated in a fixed
        order), else the SpMV followed by a dot."""
        if not hasattr(self.ops, "spmv_dot"):
            self.apply(src, dst)
            self.ops.dot(src, dst, sc, slot)
            return
        b, ops = self.block, self.ops
        if self.no_halo:
            ops.spmv_dot(self.mat, self.cfg, src, dst, src, sc, slot, False)
            return
        if src is not self._own:
            ops.copy(ops.view(self.window, self.own, b.nloc), ops.view(src, 0, b.nloc))
        sends = [(p, ops.view(src, lo - b.r0, hi - lo)) for p, lo, hi in self.plan.sends]
        recvs = [(p, ops.view(self.window, lo - b.cmin, hi - lo)) for p, lo, hi in self.plan.recvs]
        if self.parts is None:
            self.comm.exchange(sends, recvs)
            ops.spmv_dot(self.mat, self.cfg, self.window, dst, src, sc, slot, False)
            return
        token = self.comm.exchange_start(sends, recvs)
        (a, cnt, mat), rest = self.parts[0], self.parts[1:]
        ops.spmv_dot(mat, self.cfg, self.window, ops.view(dst, a, cnt), ops.view(src, a, cnt), sc, slot, False)
        self.comm.exchange_finish(token)
        for a, cnt, mat in rest:
            ops.spmv_dot(mat, self.cfg, self.window, ops.view(dst, a, cnt), ops.view(src, a, cnt), sc, slot,
                         True)

    def apply(self, src, dst):
        """dst = A_local * x, with x's local slice in ``src``."""
        b, ops = self.block, self.ops
        if self.no_halo:
            ops.spmv(self.mat, self.cfg, src, dst)
            return
        if src is not self._own:
            ops.copy(ops.view(self.window, self.own, b.nloc), ops.view(src, 0, b.nloc))
        sends = [(p, ops.view(src, lo - b.r0, hi - lo)) for p, lo, hi in self.plan.sends]
        recvs = [(p, ops.view(self.window, lo - b.cmin, hi - lo)) for p, lo, hi in self.plan.recvs]
        if self.parts is None:
            self.comm.exchange(sends, recvs)
            ops.spmv(self.mat, self.cfg, self.window, dst)
            return
        token = self.comm.exchange_start(sends, recvs)
        (a, cnt, mat), rest = self.parts[0], self.parts[1:]
        ops.spmv(mat, self.cfg, self.window, ops.view(dst, a, cnt))     # interior: own rows only
        self.comm.exchange_finish(token)
        for a, cnt, mat in rest:                                         # boundary rows
            ops.spmv(mat, self.cfg, self.window, ops.view(dst, a, cnt))


# ---------------------------------------------------------------------------
# solvers (control flow = reference _gmres_core / oracle cg)
# ---------------------------------------------------------------------------
def _finite(v: float, what: str, it: int):
    if not math.isfinite(v):
        raise SolverNumericalError(f"non-finite {what} at iteration {it}; aborting")


def _global_norm2(ops, comm, x, sc, slot: int) -> float:
    ops.dot(x, x, sc, slot)
    comm.allreduce(sc, slot, 1)
    return float(ops.read(sc, slot + 1)[slot])


class _CountingComm:
    """Counts the all-reduces a solver issues (reported per Arnoldi step)."""

    def __init__(self, comm):
        self.comm, self.allreduces = comm, 0

    def allreduce(self, sc, first, count):
        self.allreduces += 1
        self.comm.allreduce(sc, first, count)


def dist_gmres(A: DistOperator, b_local, params) -> dict:
    """Restarted GMRES over row-partitioned vectors (control flow of the
    reference's _gmres_core, solver.py:219-342) with classical Gram-Schmidt
    applied twice (CGS2) instead of modified Gram-Schmidt: MGS needs j+2
    dependent all-reduces per Arnoldi step across ranks (solver.py:294-297),
    CGS2 two — h1 = V^T w; w -= V h1 with (h2 = V^T w, ||w||^2) in the same
    sweep; w = (w - V h2) / hn with hn^2 = ||w||^2 - ||h2||^2 on the device.
    Per step: one halo exchange + local SpMV, three block sweeps over the
    basis (svb_vec_gs), two in-place all-reduces, one host read of the
    column (Givens on the host exactly as _gmres_core).  The rounding
    differs from MGS; tests hold iterations to +-1 of the MGS oracle."""
    ops = A.ops
    comm = _CountingComm(A.comm)
    m = params.restart_m
    V = ops.basis(m + 1)
    x, tmp, bvec = ops.vec(), ops.vec(), ops.vec()
    ops.upload(bvec, b_local) if isinstance(b_local, np.ndarray) else ops.copy(
        ops.view(bvec, 0, ops.n), ops.view(b_local, 0, ops.n))
    H1, H2, HN, S0 = 0, m + 1, 2 * m + 3, 2 * m + 4     # h1 | h2, ||w||^2 | hn | norms
    sc = ops.scalars(2 * m + 8)
    bnorm = math.sqrt(_global_norm2(ops, comm, bvec, sc, S0))
    hist, done = [], 0
    steps = 0
    Hh = np.zeros((m + 1, m))

    def out(conv, fin, status="ok"):
        return {"converged": conv, "iterations": done, "history": hist, "x": x, "final": fin,
                "status": status, "allreduces": comm.allreduces, "arnoldi_steps": steps,
                "orthogonalization": "CGS2 (2 all-reduces per Arnoldi step)"}

    def true_res() -> float:
        A.apply(x, tmp)
        ops.axpby(1.0, bvec, -1.0, tmp)
        return math.sqrt(_global_norm2(ops, comm, tmp, sc, S0 + 1)) / bnorm

    def update_x(j, g):
        y = np.zeros(j + 1)
        for i in range(j, -1, -1):
            y[i] = (g[i] - np.dot(Hh[i, i + 1:j + 1], y[i + 1:j + 1])) / Hh[i, i]
        ops.maxpy(V, j + 1, y, x)

    if bnorm == 0.0:
        if params.max_iters >= 1:
            hist.append(0.0)
        return out(True, 0.0)
    if params.max_iters == 0:
        return out(False, None)
    while done < params.max_iters:
        A.apply(x, tmp)
        ops.axpby(1.0, bvec, -1.0, tmp)               # r = b - A x
        beta = math.sqrt(_global_norm2(ops, comm, tmp, sc, S0 + 2))
        _finite(beta, "residual norm", done)
        if beta / bnorm <= params.tol:
            return out(True, beta / bnorm)
        ops.axpby(1.0 / beta, tmp, 0.0, V.row(0))
        Hh[:] = 0.0
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        moved, j = False, -1
        for j in range(m):
            if done >= params.max_iters:
                j -= 1
                break
            k = j + 1
            w = V.row(k)
            A.apply(V.row(j), w)
            ops.gs(ops.GS_DOT, V, k, None, 0, w, None, sc, H1)              # h1 = V^T w
            comm.allreduce(sc, H1, k)
            ops.gs(ops.GS_UPDATE, V, k, sc, H1, w, w, sc, H2)               # w -= V h1; h2, ||w||^2
            comm.allreduce(sc, H2, k + 1)
            ops.gs_hn(sc, H2, k, H2 + k, HN)
            ops.gs(ops.GS_FINISH, V, k, sc, H2, w, w, None, 0, sc, HN)      # w = (w - V h2) / hn
            steps += 1
            col = ops.read(sc, HN + 1)
            Hh[:k, j] = col[H1:H1 + k] + col[H2:H2 + k]
            hn = float(col[HN])
            _finite(hn, "Arnoldi norm", done + 1)
            for i in range(j):
                t = cs[i] * Hh[i, j] + sn[i] * Hh[i + 1, j]
                Hh[i + 1, j] = -sn[i] * Hh[i, j] + cs[i] * Hh[i + 1, j]
                Hh[i, j] = t
            d = float(np.hypot(Hh[j, j], hn))
            cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (Hh[j, j] / d, hn / d)
            Hh[j, j] = cs[j] * Hh[j, j] + sn[j] * hn
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            done += 1
            est = abs(g[j + 1]) / bnorm
            _finite(est, "residual estimate", done)
            hist.append(est)
            if hn == 0.0:
                if Hh[j, j] != 0.0:
                    update_x(j, g)
                fin = true_res()
                if fin <= params.tol:
                    return out(True, fin)
                raise StagnationError(f"Arnoldi breakdown at iteration {done} with relative "
                                      f"residual {fin:.3e} above tol {params.tol:.3e}")
            if est <= params.tol:
                update_x(j, g)
                fin = true_res()
                if fin <= params.tol:
                    return out(True, fin)
                moved = True
                break
        if j >= 0 and not moved:
            update_x(j, g)
    fin = true_res()
    return out(fin <= params.tol, fin)


def dist_cg(A: DistOperator, b_local, params) -> dict:
    """Hestenes-Stiefel CG over row-partitioned vectors (oracle/cpu_oracle.py:
    cg).  Per iteration: one halo exchange + local SpMV with the local p.Ap
    folded into the same pass (svb_vec_spmv_dot), the r update with r.r and
    alpha kept on the device (svb_dcg_rupdate), each followed by an in-place
    scalar all-reduce, then x += alpha p and p = r + beta p in one pass
    (svb_dcg_xp: 24 + 40 instead of 48 + 24 bytes per row).  The host reads
    (p.Ap, r.r) through pinned memory after the x/p pass is already
    enqueued, so the GPU keeps working while the host runs the convergence
    test; a breakdown (p.Ap = 0) stores alpha = 0 and leaves x and r
    untouched."""
    ops, comm = A.ops, A.comm
    x, r, q, bvec = ops.vec(), ops.vec(), ops.vec(), ops.vec()
    p = ops.vec() if A.no_halo else A.own_view()   # p lives in the halo window
    ops.upload(bvec, b_local) if isinstance(b_local, np.ndarray) else ops.copy(
        ops.view(bvec, 0, ops.n), ops.view(b_local, 0, ops.n))
    IALPHA = 5
    sc = ops.scalars(6)            # [rr_a, rr_b, p.Ap, ||b||^2, true residual, alpha]
    bnorm = math.sqrt(_global_norm2(ops, comm, bvec, sc, 3))
    hist, done = [], 0
    push = False                   # halo pushed by the x/p pass (PeerComm), set below

    def out(conv, fin, status="ok"):
        return {"converged": conv, "iterations": done, "history": hist, "x": x, "final": fin,
                "status": status, "halo_push": push}

    def true_res() -> float:
        A.apply(x, q)
        ops.axpby(1.0, bvec, -1.0, q)
        ops.axpby(1.0, q, 0.0, r)
        return math.sqrt(_global_norm2(ops, comm, r, sc, 4)) / bnorm

    if bnorm == 0.0:
        if params.max_iters >= 1:
            hist.append(0.0)
        return out(True, 0.0)
    if params.max_iters == 0:
        return out(False, None)
    ops.axpby(1.0, bvec, 0.0, r)
    ops.axpby(1.0, r, 0.0, p)
    cur, nxt = 0, 1
    _global_norm2(ops, comm, r, sc, cur)
    # peer-memory mode (PeerComm): the x/p pass pushes the next direction's
    # halo into the neighbours' windows, the next SpMV waits for it on the
    # device — no exchange call in the loop
    push = A.setup_push()                 # collective: every rank takes part
    pushed = False
    while done < params.max_iters:
        if pushed:
            A.apply_dot_pushed(p, q, sc, 2)
        else:
            A.apply_dot(p, q, sc, 2)          # q = A p with p.q folded into the SpMV pass
        comm.allreduce(sc, 2, 1)
        ops.cg_rupdate(sc, cur, 2, nxt, IALPHA, q, r)
        comm.allreduce(sc, nxt, 1)
        tok = ops.read_async(sc, 3)
        # x += alpha p; p = r + beta p (the p part is speculative: unused if
        # the loop stops here)
        if push:
            comm.xp_push(ops.n, sc, IALPHA, nxt, cur, r, p, x, A.push[0])
            pushed = True
        else:
            ops.cg_xp(sc, IALPHA, nxt, cur, r, p, x)
        vals = ops.read_wait(tok)
        if push or hasattr(comm, "check"):
            comm.check()                      # a timed-out peer wait raises here, not as bad numbers
        pq, rr_new = float(vals[2]), float(vals[nxt])
        _finite(pq, "curvature p.Ap", done + 1)
        if pq == 0.0:
            fin = true_res()
            if fin <= params.tol:
                return out(True, fin)
            raise StagnationError(f"CG breakdown (p.Ap = 0) at iteration {done + 1} with relative "
                                  f"residual {fin:.3e} above tol {params.tol:.3e}")
        done += 1
        est = math.sqrt(rr_new) / bnorm
        _finite(est, "residual estimate", done)
        hist.append(est)
        cur, nxt = nxt, cur
        if est <= params.tol:
            fin = true_res()                      # leaves r = b - A x
            if fin <= params.tol:
                return out(True, fin)
            ops.axpby(1.0, r, 0.0, p)
            _global_norm2(ops, comm, r, sc, cur)
            pushed = False                        # the restart's p goes out by exchange
            continue
    fin = true_res()
    return out(fin <= params.tol, fin)


# ---------------------------------------------------------------------------
# global features for the cascade (exact aggregation across ranks)
# ---------------------------------------------------------------------------
def global_features(block: LocalBlock, nrows: int, ncols: int, nnz: int, comm, local_matrix,
                    stream=None) -> FeatureVector:
    # local rows; cols window-relative.  A rank without rows contributes
    # nothing and is left out of the min (features.py:97 takes the min over
    # the matrix's rows, not over ranks)
    agg = device_aggregates(local_matrix, stream) if block.nloc > 0 else (0, 0, 0, None, 0, 0, 0)
    # span and run lengths are translation invariant; row-length stats are exact
    sums = comm.allgather_obj((agg[0], agg[1], agg[2], agg[3], agg[4], agg[5],
                               block.offsets.tolist()))
    s_r = sum(a[0] for a in sums)
    s_r2 = sum(a[1] for a in sums)
    mx = max(a[2] for a in sums)
    mn = min(a[3] for a in sums if a[3] is not None)
    span = sum(a[4] for a in sums)
    runs = sum(a[5] for a in sums)
    ndiag = len(set().union(*[set(a[6]) for a in sums]))
    return features_from_aggregates(nrows, ncols, nnz, (s_r, s_r2, mx, mn, span, runs, ndiag))


def distributed_stencil_solve(method: str, dims, offsets, weights, params, models=None,
                              initial_config: SpmvConfig | None = None, blk: "LocalBlock | None" = None,
                              timings: dict | None = None, comm_class=None):
    """Row-partitioned solve of a device-generated stencil matrix under
    torchrun (NCCL), b = A*1 (solver.py:188-193).  Each rank generates its
    z-slab on its own GPU (or reuses ``blk``); with ``models`` the cascade
    runs on the exact global features (predict-then-solve).  Returns the
    report dict (x stays on the device) and the block."""
    import time

    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    bounds = stencil_partition(dims, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    stream = device.thread_stream(0)
    if blk is None:
        blk = stencil_block(dims, offsets, weights, r0, r1, stream)
    n = blk.ncols_global
    ops, comm = CudaOps(blk.nloc, stream), peer_comm_or_base((comm_class or NcclComm)(stream), stream)
    csr = ops.local_csr(blk)
    # b = A * 1 on this rank's rows (a window of ones times the local rows),
    # outside the clock as in the reference (solver.py:355-358)
    bvec = ops.vec()
    if csr is not None:
        ones = ops.vec(blk.window)
        _lib.check(_lib.lib().svb_fill(ones.ptr, blk.window, 1.0, stream.handle))
        _lib.check(_lib.lib().svb_spmv_sequential(csr._device().handle, ones.ptr, bvec.ptr, stream.handle))
        del ones
    stream.sync()
    t0 = time.perf_counter()
    cfg = initial_config or SpmvConfig(FormatTag.CSR, Library.LIB_B)
    nnz = int(sum(comm.allgather_obj(int(csr.nnz) if csr is not None else 0)))
    if models is not None:
        from .inference import cascade_predict
        fv = global_features(blk, n, n, nnz, comm, csr, stream)
        cfg = cascade_predict(models, fv)
    t1 = time.perf_counter()
    A = DistOperator(blk, bounds, comm, ops, cfg)
    stream.sync()
    t2 = time.perf_counter()
    res = (dist_cg if method == "cg" else dist_gmres)(A, bvec, params)
    _finish_comm(comm, res)
    stream.sync()
    t3 = time.perf_counter()
    res["config"] = cfg.token()
    res["interior_rows"] = A.split
    if timings is not None:
        timings.update({"predict_s": t1 - t0, "convert_s": t2 - t1, "solve_s": t3 - t2,
                        "total_s": t3 - t0})
    return res, blk


def _finish_comm(comm, res: dict):
    """Report which collectives ran; a PeerComm surfaces a timed-out peer
    wait and unmaps the peers' buffers (collective)."""
    res["peer_collectives"] = isinstance(comm, PeerComm)
    if isinstance(comm, PeerComm):
        try:
            comm.check()
        finally:
            comm.close()


def distributed_solve(method: str, row_ptr, col_idx, values, b, params, models=None,
                      initial_config: SpmvConfig | None = None):
    """Row-partitioned solve under torchrun (NCCL).  Every rank passes the
    same global host CSR; rank r keeps rows bounds[r]:bounds[r+1].  With
    ``models`` the cascade picks the configuration from global features
    (predict-then-solve); returns (report dict, bounds)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    n = len(row_ptr) - 1
    bounds = partition_rows(row_ptr, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    blk = local_block(row_ptr, col_idx, values, r0, r1, n)
    stream = device.thread_stream(+1)
    ops, comm = CudaOps(blk.nloc, stream), peer_comm_or_base(NcclComm(stream), stream)
    cfg = initial_config or SpmvConfig(FormatTag.CSR, Library.LIB_B)
    if models is not None:
        from .inference import cascade_predict
        fv = global_features(blk, n, n, int(row_ptr[-1]), comm, ops.local_csr(blk), stream)
        cfg = cascade_predict(models, fv)
    A = DistOperator(blk, bounds, comm, ops, cfg)
    b_local = np.asarray(b[r0:r1], dtype=np.float64)
    res = (dist_cg if method == "cg" else dist_gmres)(A, b_local, params)
    _finish_comm(comm, res)
    res["config"] = cfg.token()
    res["interior_rows"] = A.split
    res["x"] = ops.fetch(res["x"])
    return res, bounds


def distributed_solve_slab(method: str, r0: int, r1: int, n: int, row_ptr, col_idx, values, b_local,
                           params, models=None, initial_config: SpmvConfig | None = None,
                           timings: dict | None = None, comm_class=None):
    """Row-partitioned solve where every rank passes only ITS OWN host slab
    (rows [r0, r1) of an n x n matrix: slab-local row_ptr, global col_idx,
    values, and b[r0:r1]) — the form a caller holding a matrix too large for
    one host (config 5: 94.7 GB as int64 CSR) uses.  Per call: the slab is
    uploaded and validated on the device, the cascade runs on the exact
    global features, the local block is converted, the solve runs, and the
    local slice of x comes back to the host.  Returns the report dict
    (``x`` = this rank's host slice)."""
    import time

    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    stream = device.thread_stream(0)
    t0 = time.perf_counter()
    blk = slab_block(r0, r1, n, row_ptr, col_idx, values, stream)
    ops, comm = CudaOps(blk.nloc, stream), peer_comm_or_base((comm_class or NcclComm)(stream), stream)
    rows = comm.allgather_obj((int(r0), int(r1)))
    bounds = np.asarray([rows[0][0]] + [r[1] for r in rows], dtype=np.int64)
    if bounds[0] != 0 or bounds[-1] != n or any(rows[k][1] != rows[k + 1][0] for k in range(world - 1)):
        raise ValueError("rank slabs must tile rows [0, n) in rank order")
    csr = ops.local_csr(blk)
    t1 = time.perf_counter()
    cfg = initial_config or SpmvConfig(FormatTag.CSR, Library.LIB_B)
    nnz = int(sum(comm.allgather_obj(int(csr.nnz) if csr is not None else 0)))
    if models is not None:
        from .inference import cascade_predict
        fv = global_features(blk, n, n, nnz, comm, csr, stream)
        cfg = cascade_predict(models, fv)
    t2 = time.perf_counter()
    A = DistOperator(blk, bounds, comm, ops, cfg)
    stream.sync()
    t3 = time.perf_counter()
    res = (dist_cg if method == "cg" else dist_gmres)(A, np.ascontiguousarray(b_local, dtype=np.float64),
                                                       params)
    _finish_comm(comm, res)
    res["x"] = ops.fetch(res["x"])
    t4 = time.perf_counter()
    res["config"] = cfg.token()
    res["interior_rows"] = A.split
    res["rank"] = rank
    if timings is not None:
        timings.update({"upload_s": t1 - t0, "predict_s": t2 - t1, "convert_s": t3 - t2,
                        "solve_s": t4 - t3, "total_s": t4 - t0})
    return res
