"""numpy restatement of the reference spmvtune hot path (CPU oracle).

TEST INFRASTRUCTURE ONLY — see ``oracle/__init__.py``.  Every function cites
the reference file:line (paths relative to ``/root/reference/pkg/src/spmvtune``)
whose observable behaviour it restates.  Matrices are plain tuples of numpy
arrays so the oracle shares no code with the product package.

Summation orders are the reference's own:
  * ``np.add.reduceat`` segment [s, e) = p[s] + pairwise(p[s+1:e])  (A.1)
  * CSR lane kernel: lane j % L sequential from 0.0, halving tree     (A.2)
  * ELL / DIA / HYB: sequential column / diagonal sweeps             (A.2)
"""
from __future__ import annotations

import math
from collections import namedtuple

import numpy as np

__all__ = [
    "OCoo", "OCsr", "OEll", "ODia", "OHyb", "OracleInapplicable",
    "DIA_CAP", "LANES", "TOKENS",
    "coo_to_csr", "csr_to_coo", "coo_to_ell", "coo_to_dia", "coo_to_hyb",
    "ell_to_coo", "dia_to_coo", "hyb_to_coo", "hyb_width", "convert", "to_coo",
    "merge_bounds", "FEATURE_ORDER",
    "spmv_sequential", "spmv", "numpy_pairwise", "segment_sum",
    "feature_aggregates", "features_from_aggregates", "features",
    "tree_predict", "cascade", "gmres", "cg", "coo_from_triplets",
]

OCoo = namedtuple("OCoo", "nrows ncols rows cols vals")
OCsr = namedtuple("OCsr", "nrows ncols ptr cols vals")
OEll = namedtuple("OEll", "nrows ncols width cols vals")   # cols/vals (nrows, width), Fortran order
ODia = namedtuple("ODia", "nrows ncols offsets data")      # data (ndiag, nrows), C order
OHyb = namedtuple("OHyb", "ell spill width")

DIA_CAP = 4096                       # formats.py:18
LANES = (2, 4, 8, 16, 32)            # kernels.py:30
TOKENS = ("COO/LibA", "CSR/LibA/2", "CSR/LibA/4", "CSR/LibA/8", "CSR/LibA/16",
          "CSR/LibA/32", "ELL/LibA", "DIA/LibA", "HYB/LibA", "COO/LibB",
          "CSR/LibB", "CSR/LibC", "ELL/LibC")  # enumerate_configs, kernels.py:92-108


class OracleInapplicable(Exception):
    """DIA above the diagonal cap (formats.py:353-356)."""


# ----------------------------------------------------------------------------
# containers / conversions (formats.py)
# ----------------------------------------------------------------------------

def coo_from_triplets(nrows, ncols, rows, cols, vals, sum_duplicates=False):
    """Lexicographic (row, col) sort, optional duplicate merge (formats.py:86-100)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.asarray(vals, np.float64)
    key = np.lexsort((cols, rows))
    rows, cols, vals = rows[key], cols[key], vals[key]
    if sum_duplicates and rows.size:
        new = np.ones(rows.size, bool)
        new[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        heads = np.nonzero(new)[0]
        vals = np.add.reduceat(vals, heads)
        rows, cols = rows[heads], cols[heads]
    return OCoo(int(nrows), int(ncols), rows, cols, vals)


def _lengths(coo: OCoo) -> np.ndarray:
    return np.bincount(coo.rows, minlength=coo.nrows).astype(np.int64)


def coo_to_csr(coo: OCoo) -> OCsr:
    """row_ptr = [0, cumsum(bincount(rows))] (formats.py:327-330)."""
    ptr = np.concatenate(([0], np.cumsum(_lengths(coo)))).astype(np.int64)
    return OCsr(coo.nrows, coo.ncols, ptr, coo.cols.copy(), coo.vals.copy())


def csr_to_coo(csr: OCsr) -> OCoo:
    """rows = repeat(arange(n), lens) (formats.py:285-287)."""
    rows = np.repeat(np.arange(csr.nrows, dtype=np.int64), np.diff(csr.ptr))
    return OCoo(csr.nrows, csr.ncols, rows, csr.cols.copy(), csr.vals.copy())


def _slot_in_row(coo: OCoo, lens):
    """Position of every entry within its row (formats.py:333-336)."""
    first = np.concatenate(([0], np.cumsum(lens)[:-1])).astype(np.int64)
    return np.arange(coo.rows.size, dtype=np.int64) - first[coo.rows]


def coo_to_ell(coo: OCoo) -> OEll:
    """Width = max row length, column-major, sentinel col = ncols (formats.py:339-348)."""
    lens = _lengths(coo)
    width = int(lens.max()) if coo.rows.size else 0
    cols = np.full((coo.nrows, width), coo.ncols, np.int64, order="F")
    vals = np.zeros((coo.nrows, width), np.float64, order="F")
    if coo.rows.size:
        slot = _slot_in_row(coo, lens)
        cols[coo.rows, slot] = coo.cols
        vals[coo.rows, slot] = coo.vals
    return OEll(coo.nrows, coo.ncols, width, cols, vals)


def coo_to_dia(coo: OCoo) -> ODia:
    """Sorted unique col-row offsets, cap 4096 (formats.py:351-361)."""
    diag = coo.cols - coo.rows
    offsets = np.unique(diag)
    if offsets.size > DIA_CAP:
        raise OracleInapplicable(f"{offsets.size} diagonals > {DIA_CAP}")
    data = np.zeros((offsets.size, coo.nrows), np.float64)
    if coo.rows.size:
        data[np.searchsorted(offsets, diag), coo.rows] = coo.vals
    return ODia(coo.nrows, coo.ncols, offsets.astype(np.int64), data)


def hyb_width(lens) -> int:
    """Smallest width covering >= ceil(2n/3) rows (formats.py:364-370)."""
    lens = np.asarray(lens)
    if lens.size == 0:
        return 0
    k = (2 * lens.size + 2) // 3
    return int(np.sort(lens)[k - 1])


def coo_to_hyb(coo: OCoo) -> OHyb:
    """ELL(w) for the first w entries of each row, row-major COO spill (formats.py:373-390)."""
    lens = _lengths(coo)
    w = hyb_width(lens)
    slot = _slot_in_row(coo, lens) if coo.rows.size else np.zeros(0, np.int64)
    keep = slot < w
    cols = np.full((coo.nrows, w), coo.ncols, np.int64, order="F")
    vals = np.zeros((coo.nrows, w), np.float64, order="F")
    if w and coo.rows.size:
        cols[coo.rows[keep], slot[keep]] = coo.cols[keep]
        vals[coo.rows[keep], slot[keep]] = coo.vals[keep]
    spill = OCoo(coo.nrows, coo.ncols, coo.rows[~keep], coo.cols[~keep], coo.vals[~keep])
    return OHyb(OEll(coo.nrows, coo.ncols, w, cols, vals), spill, w)


def ell_to_coo(ell: OEll) -> OCoo:
    """Row-major scan of the stored (non-sentinel) cells (formats.py:393-397)."""
    r, s = np.nonzero(ell.cols != ell.ncols)
    return OCoo(ell.nrows, ell.ncols, r.astype(np.int64), ell.cols[r, s].astype(np.int64),
                ell.vals[r, s].astype(np.float64))


def dia_to_coo(dia: ODia) -> OCoo:
    """In-range, non-zero diagonal cells, re-sorted (formats.py:400-416)."""
    rr, cc, vv = [], [], []
    i = np.arange(dia.nrows, dtype=np.int64)
    for k, off in enumerate(dia.offsets.tolist()):
        c = i + off
        ok = (c >= 0) & (c < dia.ncols) & (dia.data[k] != 0.0)
        rr.append(i[ok]); cc.append(c[ok]); vv.append(dia.data[k][ok])
    if not rr:
        return OCoo(dia.nrows, dia.ncols, np.zeros(0, np.int64), np.zeros(0, np.int64),
                    np.zeros(0))
    return coo_from_triplets(dia.nrows, dia.ncols, np.concatenate(rr),
                             np.concatenate(cc), np.concatenate(vv))


def hyb_to_coo(h: OHyb) -> OCoo:
    """ELL part plus spill, re-sorted (formats.py:292-298)."""
    e = ell_to_coo(h.ell)
    return coo_from_triplets(h.ell.nrows, h.ell.ncols,
                             np.concatenate([e.rows, h.spill.rows]),
                             np.concatenate([e.cols, h.spill.cols]),
                             np.concatenate([e.vals, h.spill.vals]))


def to_coo(m) -> OCoo:
    if isinstance(m, OCoo):
        return m
    if isinstance(m, OCsr):
        return csr_to_coo(m)
    if isinstance(m, OEll):
        return ell_to_coo(m)
    if isinstance(m, ODia):
        return dia_to_coo(m)
    if isinstance(m, OHyb):
        return hyb_to_coo(m)
    raise TypeError(type(m))


def convert(m, target: str):
    """Hub conversion through COO (formats.py:302-320)."""
    coo = to_coo(m)
    return {"COO": lambda c: c, "CSR": coo_to_csr, "ELL": coo_to_ell,
            "DIA": coo_to_dia, "HYB": coo_to_hyb}[target](coo)


# ----------------------------------------------------------------------------
# summation primitives
# ----------------------------------------------------------------------------

def numpy_pairwise(a) -> float:
    """numpy's float64 pairwise sum (numpy/_core/src/umath/loops_utils.h.src),
    restated in pure Python.  Used to document/verify the order the CUDA
    kernels implement; ``segment_sum`` below is the reduceat composition."""
    a = [float(v) for v in a]

    def pw(lo, n):
        if n < 8:
            r = -0.0
            for i in range(n):
                r += a[lo + i]
            return r
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for k in range(8):
                    r[k] += a[lo + i + k]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return pw(lo, n2) + pw(lo + n2, n - n2)

    return pw(0, len(a))


def segment_sum(p, s, e) -> float:
    """``np.add.reduceat`` over one segment [s, e): p[s] + pairwise(p[s+1:e])."""
    if e - s == 1:
        return float(p[s])
    return float(p[s]) + numpy_pairwise(p[s + 1:e])


def spmv_sequential(csr: OCsr, x) -> np.ndarray:
    """Row-wise ascending-column accumulation from 0.0 (formats.py:419-435),
    vectorised over rows by in-row position (same per-row order)."""
    x = np.asarray(x, np.float64)
    lens = np.diff(csr.ptr)
    y = np.zeros(csr.nrows)
    for j in range(int(lens.max()) if lens.size else 0):
        live = np.nonzero(lens > j)[0]
        k = csr.ptr[live] + j
        y[live] += csr.vals[k] * x[csr.cols[k]]
    return y


# ----------------------------------------------------------------------------
# the 13 SpMV kernels (kernels.py:146-312)
# ----------------------------------------------------------------------------

def _row_runs(rows):
    head = np.ones(rows.size, bool)
    head[1:] = rows[1:] != rows[:-1]
    starts = np.nonzero(head)[0]
    return starts, rows[starts]


def _coo_liba(m: OCoo, x, y):                       # kernels.py:146-153
    if m.rows.size:
        p = m.vals * x[m.cols]
        starts, rws = _row_runs(m.rows)
        y[rws] = np.add.reduceat(p, starts)


def _coo_libb(m: OCoo, x, y):                       # kernels.py:156-164
    if m.rows.size:
        order = np.random.default_rng().permutation(m.rows.size)
        np.add.at(y, m.rows[order], m.vals[order] * x[m.cols[order]])


def _csr_lanes(m: OCsr, x, y, L):                   # kernels.py:167-189
    if not m.cols.size:
        return
    lens = np.diff(m.ptr)
    acc = np.zeros((m.nrows, L))
    for j in range(int(lens.max())):
        live = np.nonzero(lens > j)[0]
        k = m.ptr[live] + j
        acc[live, j % L] += m.vals[k] * x[m.cols[k]]
    h = L
    while h > 1:
        h //= 2
        acc[:, :h] += acc[:, h:2 * h]
    y[:] = acc[:, 0]


def _csr_libb(m: OCsr, x, y):                       # kernels.py:192-199
    if m.cols.size:
        p = m.vals * x[m.cols]
        ne = np.diff(m.ptr) > 0
        y[ne] = np.add.reduceat(p, m.ptr[:-1][ne])


def merge_bounds(nnz: int, workers: int) -> np.ndarray:
    """Chunk edges of the LibC merge-path kernel (kernels.py:209-210)."""
    return np.linspace(0, nnz, min(workers, nnz) + 1, dtype=np.int64)


def _csr_libc(m: OCsr, x, y, workers):              # kernels.py:202-223
    nnz = m.cols.size
    if not nnz:
        return
    p = m.vals * x[m.cols]
    b = merge_bounds(nnz, workers)
    for c in range(b.size - 1):
        e0, e1 = int(b[c]), int(b[c + 1])
        if e0 == e1:
            continue
        r0 = int(np.searchsorted(m.ptr, e0, side="right")) - 1
        r1 = int(np.searchsorted(m.ptr, e1, side="left"))
        lo = np.maximum(m.ptr[r0:r1], e0)
        cnt = np.diff(np.append(lo, e1))
        ne = np.nonzero(cnt > 0)[0]
        y[r0 + ne] += np.add.reduceat(p[e0:e1], lo[ne] - e0)


def _ell_sweep(m: OEll, x, y):                      # kernels.py:226-233
    if m.width:
        xe = np.append(x, 0.0)
        for k in range(m.width):
            y += m.vals[:, k] * xe[m.cols[:, k]]


def _ell_strided(m: OEll, x, y, workers):           # kernels.py:236-248
    if m.width:
        xe = np.append(x, 0.0)
        S = min(workers, m.width)
        for w in range(S):
            part = np.zeros(m.nrows)
            for k in range(w, m.width, S):
                part += m.vals[:, k] * xe[m.cols[:, k]]
            y += part


def _dia_sweep(m: ODia, x, y):                      # kernels.py:251-260
    for k, off in enumerate(m.offsets.tolist()):
        lo, hi = max(0, -off), min(m.nrows, m.ncols - off)
        if lo < hi:
            y[lo:hi] += m.data[k, lo:hi] * x[lo + off:hi + off]


def _hyb(m: OHyb, x, y):                            # kernels.py:263-271
    _ell_sweep(m.ell, x, y)
    s = m.spill
    if s.rows.size:
        p = s.vals * x[s.cols]
        starts, rws = _row_runs(s.rows)
        y[rws] += np.add.reduceat(p, starts)


def spmv(token: str, m, x, workers: int = 4) -> np.ndarray:
    """Dispatch one of the 13 configurations (kernels.py:274-312)."""
    x = np.ascontiguousarray(x, np.float64)
    nrows = m.ell.nrows if isinstance(m, OHyb) else m.nrows
    y = np.zeros(nrows)
    parts = token.split("/")
    fmt, lib = parts[0], parts[1]
    if fmt == "COO":
        (_coo_liba if lib == "LibA" else _coo_libb)(m, x, y)
    elif fmt == "CSR":
        if lib == "LibA":
            _csr_lanes(m, x, y, int(parts[2]))
        elif lib == "LibB":
            _csr_libb(m, x, y)
        else:
            _csr_libc(m, x, y, workers)
    elif fmt == "ELL":
        if lib == "LibA":
            _ell_sweep(m, x, y)
        else:
            _ell_strided(m, x, y, workers)
    elif fmt == "DIA":
        _dia_sweep(m, x, y)
    else:
        _hyb(m, x, y)
    return y


# ----------------------------------------------------------------------------
# features (features.py:68-156)
# ----------------------------------------------------------------------------

FEATURE_ORDER = ("nrows", "ncols", "nnz", "density", "mean", "sd", "cov", "max",
                 "min", "maxavg", "distavg", "clusteravg", "fill", "ndiag",
                 "diagfill")                       # features.py:19-21


def feature_aggregates(csr: OCsr) -> dict:
    """The seven exact integer aggregates the 15 features derive from."""
    lens = np.diff(csr.ptr)
    n = csr.nrows
    agg = {"sum_r": int(lens.sum()), "sum_r2": int((lens * lens).sum()),
           "max_r": int(lens.max()) if n else 0,
           "min_r": int(lens.min()) if n else 0}
    ne = lens > 0
    if csr.cols.size:
        first = csr.cols[csr.ptr[:-1][ne]]
        last = csr.cols[csr.ptr[1:][ne] - 1]
        agg["span"] = int((last - first).sum())
        rows = np.repeat(np.arange(n, dtype=np.int64), lens)
        cont = np.zeros(csr.cols.size, bool)
        cont[1:] = (np.diff(csr.cols) == 1) & (np.diff(rows) == 0)
        heads = np.nonzero(~cont)[0]
        runlen = np.diff(np.append(heads, csr.cols.size))
        best = np.zeros(n, np.int64)
        np.maximum.at(best, rows[heads], runlen)
        agg["runs"] = int(best.sum())
        agg["ndiag"] = int(np.unique(csr.cols - rows).size)
    else:
        agg["span"] = agg["runs"] = agg["ndiag"] = 0
    return agg


def features_from_aggregates(nrows, ncols, nnz, a: dict) -> list:
    """The float formulas of features.py:103-110 and 147-150, verbatim order."""
    min_r = a["min_r"] or 0
    density = nnz / (nrows * ncols)
    mean = nnz / nrows
    sd = float(np.sqrt(max(a["sum_r2"] / nrows - mean * mean, 0.0)))
    cov = sd / mean if mean > 0 else 0.0
    maxavg = a["max_r"] - mean
    fill = nrows * a["max_r"] / nnz if nnz > 0 else 0.0
    distavg = a["span"] / nrows
    clusteravg = a["runs"] / nrows
    diagfill = nrows * a["ndiag"] / nnz if nnz > 0 else 0.0
    return [nrows, ncols, nnz, density, mean, sd, cov, float(a["max_r"]),
            float(min_r), maxavg, distavg, clusteravg, fill, float(a["ndiag"]),
            diagfill]


def features(csr: OCsr) -> list:
    return features_from_aggregates(csr.nrows, csr.ncols, int(csr.cols.size),
                                    feature_aggregates(csr))


# ----------------------------------------------------------------------------
# cascade inference (inference.py:108-119, 283-324; docs/model_schema.md)
# ----------------------------------------------------------------------------

def tree_predict(doc: dict, x) -> tuple[str, list]:
    """Per-class leaf sums in list order, `<=` goes left, ties -> lowest index."""
    x = [float(v) for v in x]
    sums = []
    for class_trees in doc["trees"]:
        total = 0.0
        for node in class_trees:
            while "score" not in node:
                node = node["left"] if x[node["feature_index"]] <= node["threshold"] \
                    else node["right"]
            total += float(node["score"])
        sums.append(total)
    best = 0
    for k in range(1, len(sums)):
        if sums[k] > sums[best]:
            best = k
    return doc["classes"][best], sums


def cascade(models: dict, x) -> list[str]:
    """Staged decisions as implied-config tokens; last one is final (inference.py:283-324)."""
    fmt, _ = tree_predict(models["FORMAT"], x)
    if fmt in ("DIA", "HYB"):
        return [f"{fmt}/LibA"]
    out = [f"{fmt}/LibA/32" if fmt == "CSR" else f"{fmt}/LibA"]   # implied_config, inference.py:231-241
    lib, _ = tree_predict(models[{"COO": "COO-LIB", "CSR": "CSR-LIB", "ELL": "ELL-LIB"}[fmt]], x)
    if fmt == "CSR" and lib == "LibA":
        out.append("CSR/LibA/32")
        lane, _ = tree_predict(models["CSR-TPV"], x)
        out.append(f"CSR/LibA/{lane}")
    else:
        out.append(f"{fmt}/{lib}")
    return out


# ----------------------------------------------------------------------------
# Krylov solvers
# ----------------------------------------------------------------------------

def _back_substitute(H, g, j, V):
    """solver.py:211-216."""
    y = np.zeros(j + 1)
    for i in range(j, -1, -1):
        y[i] = (g[i] - np.dot(H[i, i + 1:j + 1], y[i + 1:j + 1])) / H[i, i]
    return V[:j + 1].T @ y


def gmres(matvec, b, restart=30, tol=1e-8, max_iters=1000, on_iteration=None) -> dict:
    """Restarted MGS-GMRES with Givens rotations and explicit-residual
    confirmation, restating solver.py:219-342 without the mailbox.

    Returns dict(converged, iterations, history, x, final, status) where
    status is 'ok' / 'stagnation' / 'nonfinite'."""
    n = b.size
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    hist = []
    done = 0

    def out(conv, fin, status="ok"):
        return dict(converged=conv, iterations=done, history=hist, x=x, final=fin,
                    status=status)

    if bnorm == 0.0:
        if max_iters >= 1:
            hist.append(0.0)
        return out(True, 0.0)
    if max_iters == 0:
        return out(False, None)
    while done < max_iters:
        r = b - matvec(x)
        beta = float(np.linalg.norm(r))
        if not math.isfinite(beta):
            return out(False, None, "nonfinite")
        if beta / bnorm <= tol:
            return out(True, beta / bnorm)
        V = np.empty((restart + 1, n))
        V[0] = r / beta
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        moved = False
        j = -1
        for j in range(restart):
            if done >= max_iters:
                j -= 1
                break
            w = matvec(V[j])
            for i in range(j + 1):
                H[i, j] = float(np.dot(V[i], w))
                w -= H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            if not math.isfinite(hn):
                return out(False, None, "nonfinite")
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = float(np.hypot(H[j, j], hn))
            cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (H[j, j] / d, hn / d)
            H[j, j] = cs[j] * H[j, j] + sn[j] * hn
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            done += 1
            est = abs(g[j + 1]) / bnorm
            if not math.isfinite(est):
                return out(False, None, "nonfinite")
            hist.append(est)
            if on_iteration is not None:
                on_iteration(done, j)
            if hn == 0.0:
                if H[j, j] != 0.0:
                    x = x + _back_substitute(H, g, j, V)
                fin = float(np.linalg.norm(b - matvec(x))) / bnorm
                return out(True, fin) if fin <= tol else out(False, fin, "stagnation")
            if est <= tol:
                x = x + _back_substitute(H, g, j, V)
                fin = float(np.linalg.norm(b - matvec(x))) / bnorm
                if fin <= tol:
                    return out(True, fin)
                moved = True
                break
            V[j + 1] = w / hn
        if j >= 0 and not moved:
            x = x + _back_substitute(H, g, j, V)
    fin = float(np.linalg.norm(b - matvec(x))) / bnorm
    return out(fin <= tol, fin)


def cg(matvec, b, tol=1e-8, max_iters=1000, dot=None) -> dict:
    """Hestenes–Stiefel CG.  The reference has NO CG; this is the
    new oracle SURVEY.md §8c specifies: x0 = 0, one matvec per iteration,
    recurrence residual ||r||/||b|| as the per-iteration estimate, explicit
    residual confirmation on convergence (mirroring GMRES, solver.py:328-336),
    restart from the true residual when the estimate drifted."""
    n = b.size
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    hist = []
    done = 0

    def out(conv, fin, status="ok"):
        return dict(converged=conv, iterations=done, history=hist, x=x, final=fin,
                    status=status)

    if bnorm == 0.0:
        if max_iters >= 1:
            hist.append(0.0)
        return out(True, 0.0)
    if max_iters == 0:
        return out(False, None)
    if dot is None:       # the reference's inner product (BLAS ddot via np.dot)
        dot = np.dot
    r = b.copy()
    p = r.copy()
    rr = float(dot(r, r))
    while done < max_iters:
        q = matvec(p)
        pq = float(dot(p, q))
        if not math.isfinite(pq):
            return out(False, None, "nonfinite")
        if pq == 0.0:
            fin = float(np.linalg.norm(b - matvec(x))) / bnorm
            return out(True, fin) if fin <= tol else out(False, fin, "stagnation")
        alpha = rr / pq
        x = x + alpha * p
        r = r - alpha * q
        rr_new = float(dot(r, r))
        done += 1
        est = math.sqrt(rr_new) / bnorm
        if not math.isfinite(est):
            return out(False, None, "nonfinite")
        hist.append(est)
        if est <= tol:
            r = b - matvec(x)
            fin = float(np.linalg.norm(r)) / bnorm
            if fin <= tol:
                return out(True, fin)
            p = r.copy()
            rr = float(dot(r, r))
            continue
        p = r + (rr_new / rr) * p
        rr = rr_new
    fin = float(np.linalg.norm(b - matvec(x))) / bnorm
    return out(fin <= tol, fin)
