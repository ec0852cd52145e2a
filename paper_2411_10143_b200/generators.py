"""Vectorised synthetic-matrix generators for the BASELINE configurations.

Host (numpy) builders return ``(nrows, ncols, row_ptr, col_idx, values)``
CSR triples with int64 indices, columns strictly increasing per row — the
exact layout ``CsrMatrix`` (formats.py:103-146 in the reference) accepts.
Large stencils (configs 2 and 5) are also generated directly on the device
by ``formats.CsrMatrix.stencil`` (csrc/generate.cu), which never touches host
memory; both produce identical arrays (tests/test_gpu_generate.py).

The stencil structures follow SURVEY.md §8(d): ``poisson2d`` mirrors the
reference test helper (tests/helpers.py:42-64), ``convdiff9`` is the
nonsymmetric 9-point convection-diffusion operator and ``laplace27`` the
3-D 27-point Laplacian.
"""
from __future__ import annotations

import numpy as np

__all__ = ["poisson2d", "convdiff9", "laplace27", "powerlaw_spd", "banded",
           "stencil_csr"]


def stencil_csr(dims, offsets, weights):
    """CSR of a constant-coefficient stencil on a Cartesian grid.

    ``dims`` is the grid shape with the fastest axis LAST (row index
    ``i = ((z * ny) + y) * nx + x``); ``offsets`` is a list of per-axis
    displacement tuples and ``weights`` their coefficients.  Neighbours that
    fall outside the grid are dropped (Dirichlet boundary)."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    strides = np.cumprod((1,) + dims[::-1][:-1])[::-1]
    lin = [int(np.dot(o, strides)) for o in offsets]
    order = np.argsort(lin, kind="stable")        # ascending column offset
    offsets = [offsets[k] for k in order]
    weights = [float(weights[k]) for k in order]
    lin = [lin[k] for k in order]
    coords = np.indices(dims).reshape(len(dims), -1)
    masks = []
    for off in offsets:
        ok = np.ones(n, bool)
        for ax, d in enumerate(off):
            c = coords[ax] + d
            ok &= (c >= 0) & (c < dims[ax])
        masks.append(ok)
    masks = np.stack(masks)                        # (nstencil, n)
    lens = masks.sum(axis=0).astype(np.int64)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    base = np.arange(n, dtype=np.int64)
    cols2d = base[None, :] + np.asarray(lin, np.int64)[:, None]
    vals2d = np.broadcast_to(np.asarray(weights)[:, None], masks.shape)
    # row-major flattening of the (row, stencil-slot) table keeps each row's
    # columns ascending because the stencil slots are sorted by offset
    col_idx = cols2d.T[masks.T]
    values = np.ascontiguousarray(vals2d.T[masks.T], dtype=np.float64)
    return n, n, row_ptr, col_idx.astype(np.int64), values


def poisson2d(nx: int):
    """5-point Laplacian, diag 4 / off -1 (config 1)."""
    offs = [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)]
    w = [4.0, -1.0, -1.0, -1.0, -1.0]
    return stencil_csr((nx, nx), offs, w)


def convdiff9(nx: int, diag: float = 8.5, beta: float = 0.25):
    """Nonsymmetric 9-point convection-diffusion (config 2): centre ``diag``,
    neighbour (dy, dx) weight ``-1 - beta*(dx + dy)``."""
    offs, w = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dy, dx))
            w.append(diag if (dx, dy) == (0, 0) else -1.0 - beta * (dx + dy))
    return stencil_csr((nx, nx), offs, w)


def laplace27(n: int):
    """3-D 27-point Laplacian, diag 26 / off -1 (config 5)."""
    offs, w = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dz, dy, dx))
                w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
    return stencil_csr((n, n, n), offs, w)


def powerlaw_spd(n: int, alpha: float = 2.1, mean_deg: float = 7.0, seed: int = 0):
    """Symmetric diagonally-dominant matrix with Pareto(alpha) out-degrees
    (config 3): uniform random targets, symmetrised, off-diagonal values
    -U(0.1, 1), diagonal = sum |off-diagonal| + 1."""
    rng = np.random.default_rng(seed)
    xm = mean_deg * (alpha - 1.0) / alpha
    deg = np.floor(xm * (1.0 + rng.pareto(alpha, size=n))).astype(np.int64)
    deg = np.minimum(deg, n - 1)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    dst = rng.integers(0, n, size=src.size, dtype=np.int64)
    keep = src != dst
    a, b = np.minimum(src[keep], dst[keep]), np.maximum(src[keep], dst[keep])
    key = np.unique(a * n + b)                     # undirected edge set
    a, b = key // n, key % n
    w = -rng.uniform(0.1, 1.0, size=key.size)
    rows = np.concatenate([a, b, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([b, a, np.arange(n, dtype=np.int64)])
    absum = np.bincount(a, weights=-w, minlength=n) + np.bincount(b, weights=-w, minlength=n)
    vals = np.concatenate([w, w, absum + 1.0])
    order = np.argsort(rows * n + cols, kind="stable")
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return n, n, row_ptr, cols, np.ascontiguousarray(vals)


def powerlaw_spd_device(n: int, alpha: float = 2.1, mean_deg: float = 7.0, seed: int = 0):
    """``powerlaw_spd`` built on the device: the same random draws in the
    same order and the same numpy bincount sums for the diagonal, but the
    two sorts (undirected-edge dedupe, row-major order) run as device radix
    sorts (CooMatrix.from_triplets_device) instead of np.unique / argsort —
    50+ s on the host at config 3's 8 M rows.  Returns a device CsrMatrix
    whose arrays equal powerlaw_spd's bit for bit (tests/test_gpu_scale.py)."""
    from .formats import CooMatrix, FormatTag, convert
    rng = np.random.default_rng(seed)
    xm = mean_deg * (alpha - 1.0) / alpha
    deg = np.floor(xm * (1.0 + rng.pareto(alpha, size=n))).astype(np.int64)
    deg = np.minimum(deg, n - 1)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    dst = rng.integers(0, n, size=src.size, dtype=np.int64)
    keep = src != dst
    a, b = np.minimum(src[keep], dst[keep]), np.maximum(src[keep], dst[keep])
    del src, dst, keep
    edges = CooMatrix.from_triplets_device(n, n, a, b, np.zeros(a.size), sum_duplicates=True)
    del a, b
    a, b = edges.rows, edges.cols                  # ascending (a, b) == np.unique(a*n+b) order
    del edges
    w = -rng.uniform(0.1, 1.0, size=a.size)
    absum = np.bincount(a, weights=-w, minlength=n) + np.bincount(b, weights=-w, minlength=n)
    diag = np.arange(n, dtype=np.int64)
    coo = CooMatrix.from_triplets_device(n, n, np.concatenate([a, b, diag]), np.concatenate([b, a, diag]),
                                         np.concatenate([w, w, absum + 1.0]))
    return convert(coo, FormatTag.CSR)


def banded(n: int, offsets, seed: int = 0, diagonal_boost: float = 0.0):
    """Positive values on the given diagonals (tests/helpers.py:67-84 shape)."""
    rng = np.random.default_rng(seed)
    offsets = sorted(set(int(o) for o in offsets))
    rows, cols, vals = [], [], []
    i = np.arange(n, dtype=np.int64)
    for off in offsets:
        c = i + off
        ok = (c >= 0) & (c < n)
        v = rng.uniform(0.5, 1.5, size=int(ok.sum()))
        if off == 0:
            v = v + diagonal_boost
        rows.append(i[ok]); cols.append(c[ok]); vals.append(v)
    rows = np.concatenate(rows); cols = np.concatenate(cols); vals = np.concatenate(vals)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return n, n, row_ptr, cols, vals
