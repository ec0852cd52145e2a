"""Sparse containers for the five storage layouts, resident on the B200.

Drop-in for the reference ``spmvtune.formats`` (formats.py:1-435): same class
names, constructor signatures, validation messages and read-only array
attributes.  The difference is where the data lives: every container owns an
immutable device handle (``svb_matrix``) and the numpy attributes are a lazy
host mirror —

* containers built from host arrays validate them like the reference and
  upload on first device use;
* containers produced by ``convert`` (or the on-device generators) exist
  only on the device until an attribute such as ``row_ptr`` is read, at
  which point that array is downloaded once and frozen.

``convert`` runs entirely on the GPU (csrc/convert.cu) and returns arrays
bit-identical to the reference's.
"""
from __future__ import annotations

import threading
from enum import Enum

import numpy as np

from . import _lib
from .errors import FormatInapplicableError  # noqa: F401  (re-export parity)

DIA_OFFSET_CAP = 4096          # formats.py:18
# Device memory guard for ELL (absent in the reference, SURVEY.md §7 hard
# part 4): a padded layout may use at most max(2^26, 8 * nnz) cells, so a
# power-law matrix whose longest row is 200x the mean is "inapplicable"
# instead of allocating tens of GB of padding.
ELL_MIN_CELLS = 1 << 26
ELL_PAD_FACTOR = 8


class FormatTag(str, Enum):
    COO = "COO"
    CSR = "CSR"
    ELL = "ELL"
    DIA = "DIA"
    HYB = "HYB"


_TAG_CODE = {FormatTag.COO: _lib.COO, FormatTag.CSR: _lib.CSR, FormatTag.ELL: _lib.ELL,
             FormatTag.DIA: _lib.DIA, FormatTag.HYB: _lib.HYB}


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


def _index_vector(a, what: str) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.int64)
    if out.ndim != 1:
        raise ValueError(f"{what} must be one-dimensional")
    return out


def _value_vector(a, what: str) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if out.ndim != 1:
        raise ValueError(f"{what} must be one-dimensional")
    if out.size and not np.isfinite(out).all():
        raise ValueError(f"{what} contains non-finite values")
    return out


class DeviceMatrix:
    """Owner of one ``svb_matrix*``; destroyed with the Python object."""

    __slots__ = ("handle", "info", "__weakref__")

    def __init__(self, handle: int):
        self.handle = handle
        info = _lib.MatrixInfo()
        _lib.check(_lib.load().svb_matrix_info_get(handle, info))
        self.info = info

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.load().svb_matrix_destroy(h)
            except Exception:
                pass

    def download(self, which: int, count: int, dtype) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        if count:
            _lib.check(_lib.lib().svb_matrix_download(self.handle, which, out.ctypes.data, None))
        return out


def _new_handle(fn, *args) -> DeviceMatrix:
    import ctypes
    h = ctypes.c_void_p()
    _lib.check(fn(*args, ctypes.byref(h)))
    return DeviceMatrix(h.value)


class _Resident:
    """Shared machinery: lazy upload of host arrays / lazy download of device
    arrays, guarded so concurrent solver and advisor threads see one copy."""

    _tag: FormatTag

    def _init_resident(self, dev: DeviceMatrix | None = None):
        self._dev = dev
        self._host = {}
        self._lock = threading.RLock()

    def _device(self) -> DeviceMatrix:
        if self._dev is None:
            with self._lock:
                if self._dev is None:
                    self._dev = self._upload()
        return self._dev

    def _get(self, key, fetch):
        arr = self._host.get(key)
        if arr is None:
            with self._lock:
                arr = self._host.get(key)
                if arr is None:
                    arr = _frozen(fetch())
                    self._host[key] = arr
        return arr

    @property
    def device_bytes(self) -> int:
        return int(self._device().info.device_bytes)

    def __getstate__(self):
        raise TypeError("device-resident matrices are not picklable; pass host arrays instead")


class CooMatrix(_Resident):
    """Coordinate triplets sorted row-major with no duplicate coordinates
    (formats.py:50-100)."""

    _tag = FormatTag.COO

    def __init__(self, nrows, ncols, rows, cols, values):
        if nrows < 1 or ncols < 1:
            raise ValueError("matrix dimensions must be positive")
        self.nrows, self.ncols = int(nrows), int(ncols)
        r = _index_vector(rows, "rows")
        c = _index_vector(cols, "cols")
        v = _value_vector(values, "values")
        if not (r.size == c.size == v.size):
            raise ValueError("rows, cols, values must have equal length")
        if r.size:
            if r.min() < 0 or r.max() >= self.nrows:
                raise ValueError("row index out of range")
            if c.min() < 0 or c.max() >= self.ncols:
                raise ValueError("column index out of range")
            step = np.diff(r)
            if (step < 0).any():
                raise ValueError("entries not sorted by row")
            if (np.diff(c)[step == 0] <= 0).any():
                raise ValueError("entries not strictly sorted by column within rows")
        self._nnz = int(v.size)
        self._init_resident()
        self._host = {"rows": _frozen(r), "cols": _frozen(c), "values": _frozen(v)}

    @classmethod
    def _wrap(cls, dev: DeviceMatrix):
        self = cls.__new__(cls)
        self.nrows, self.ncols = int(dev.info.nrows), int(dev.info.ncols)
        self._nnz = int(dev.info.nnz)
        self._init_resident(dev)
        return self

    def _upload(self):
        return _new_handle(_lib.lib().svb_coo_create, self.nrows, self.ncols, self._nnz,
                           self.rows.ctypes.data, self.cols.ctypes.data, self.values.ctypes.data, None)

    rows = property(lambda s: s._get("rows", lambda: s._dev.download(_lib.ARR_ROWS, s._nnz, np.int64)))
    cols = property(lambda s: s._get("cols", lambda: s._dev.download(_lib.ARR_COLS, s._nnz, np.int64)))
    values = property(lambda s: s._get("values", lambda: s._dev.download(_lib.ARR_VALS, s._nnz, np.float64)))

    @property
    def nnz(self) -> int:
        return self._nnz

    @classmethod
    def from_triplets(cls, nrows, ncols, rows, cols, values, *, sum_duplicates=False):
        """Sort unsorted triplets row-major; optionally merge duplicate
        coordinates by summation (formats.py:86-100)."""
        r = _index_vector(rows, "rows")
        c = _index_vector(cols, "cols")
        v = _value_vector(values, "values")
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        if sum_duplicates and r.size:
            head = np.ones(r.size, dtype=bool)
            head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            first = np.flatnonzero(head)
            v = np.add.reduceat(v, first)
            r, c = r[first], c[first]
        return cls(nrows, ncols, r, c, v)


    @classmethod
    def from_triplets_device(cls, nrows, ncols, rows, cols, values, *, sum_duplicates=False):
        """``from_triplets`` with the sort (stable radix sort) and the
        duplicate merge (np.add.reduceat order) on the device
        (svb_coo_from_triplets); the result stays device-resident."""
        r = np.ascontiguousarray(rows, dtype=np.int64)
        c = np.ascontiguousarray(cols, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        if not (r.size == c.size == v.size):
            raise ValueError("rows, cols and values must have equal length")
        dev = _new_handle(_lib.lib().svb_coo_from_triplets, int(nrows), int(ncols), int(r.size),
                          r.ctypes.data, c.ctypes.data, v.ctypes.data, 1 if sum_duplicates else 0, None)
        return cls._wrap(dev)


class CsrMatrix(_Resident):
    """Compressed sparse rows; columns strictly increasing within each row
    (formats.py:103-146)."""

    _tag = FormatTag.CSR

    def __init__(self, nrows, ncols, row_ptr, col_idx, values):
        if nrows < 1 or ncols < 1:
            raise ValueError("matrix dimensions must be positive")
        self.nrows, self.ncols = int(nrows), int(ncols)
        p = _index_vector(row_ptr, "row_ptr")
        c = _index_vector(col_idx, "col_idx")
        v = _value_vector(values, "values")
        if p.size != self.nrows + 1:
            raise ValueError("row_ptr must have nrows+1 entries")
        if p[0] != 0 or p[-1] != v.size:
            raise ValueError("row_ptr endpoints must be 0 and nnz")
        if (np.diff(p) < 0).any():
            raise ValueError("row_ptr must be non-decreasing")
        if c.size != v.size:
            raise ValueError("col_idx and values must have equal length")
        if c.size:
            if c.min() < 0 or c.max() >= self.ncols:
                raise ValueError("column index out of range")
            same_row = np.ones(c.size - 1, dtype=bool)
            cut = p[1:-1]
            cut = cut[(cut > 0) & (cut < c.size)]
            same_row[cut - 1] = False
            if (np.diff(c)[same_row] <= 0).any():
                raise ValueError("columns not strictly increasing within a row")
        self._nnz = int(v.size)
        self._init_resident()
        self._host = {"row_ptr": _frozen(p), "col_idx": _frozen(c), "values": _frozen(v)}

    @classmethod
    def _wrap(cls, dev: DeviceMatrix):
        self = cls.__new__(cls)
        self.nrows, self.ncols = int(dev.info.nrows), int(dev.info.ncols)
        self._nnz = int(dev.info.nnz)
        self._init_resident(dev)
        return self

    @classmethod
    def stencil(cls, dims, offsets, weights):
        """Generate a constant-coefficient stencil matrix directly on the
        device (csrc/generate.cu); identical to generators.stencil_csr."""
        import ctypes
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        offs = np.ascontiguousarray(offsets, dtype=np.int32).reshape(-1)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        L = _lib.lib()
        dev = _new_handle(L.svb_csr_stencil, int(dims.size),
                          dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(w.size),
                          offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                          w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), None)
        return cls._wrap(dev)

    def _upload(self):
        return _new_handle(_lib.lib().svb_csr_create, self.nrows, self.ncols, self._nnz,
                           self.row_ptr.ctypes.data, self.col_idx.ctypes.data,
                           self.values.ctypes.data, None)

    row_ptr = property(lambda s: s._get("row_ptr", lambda: s._dev.download(
        _lib.ARR_ROW_PTR, s.nrows + 1, np.int64)))
    col_idx = property(lambda s: s._get("col_idx", lambda: s._dev.download(_lib.ARR_COLS, s._nnz, np.int64)))
    values = property(lambda s: s._get("values", lambda: s._dev.download(_lib.ARR_VALS, s._nnz, np.float64)))

    @property
    def nnz(self) -> int:
        return self._nnz

    @property
    def row_lengths(self) -> np.ndarray:
        return np.diff(self.row_ptr)


class EllMatrix(_Resident):
    """Fixed-width padded rows in column-major order (formats.py:149-186);
    padding cells hold column ``ncols`` and value 0."""

    _tag = FormatTag.ELL

    def __init__(self, nrows, ncols, width, col_idx, values):
        if nrows < 1 or ncols < 1:
            raise ValueError("matrix dimensions must be positive")
        if width < 0:
            raise ValueError("width must be non-negative")
        self.nrows, self.ncols, self.width = int(nrows), int(ncols), int(width)
        c = np.asfortranarray(col_idx, dtype=np.int64)
        v = np.asfortranarray(values, dtype=np.float64)
        shape = (self.nrows, self.width)
        if c.shape != shape or v.shape != shape:
            raise ValueError("col_idx and values must be nrows x width")
        if self.width:
            if c.min() < 0 or c.max() > self.ncols:
                raise ValueError("column index out of range")
            if (v[c == self.ncols] != 0.0).any():
                raise ValueError("padding cells must hold value 0")
            if not np.isfinite(v).all():
                raise ValueError("values contain non-finite entries")
        self._init_resident()
        self._host = {"col_idx": _frozen(c), "values": _frozen(v)}

    @classmethod
    def _wrap(cls, dev: DeviceMatrix):
        self = cls.__new__(cls)
        self.nrows, self.ncols = int(dev.info.nrows), int(dev.info.ncols)
        self.width = int(dev.info.width)
        self._init_resident(dev)
        return self

    def _upload(self):
        # column-major (nrows x width) == row-major (width x nrows) buffer
        c = np.ascontiguousarray(self.col_idx.T)
        v = np.ascontiguousarray(self.values.T)
        return _new_handle(_lib.lib().svb_ell_create, self.nrows, self.ncols, self.width,
                           c.ctypes.data, v.ctypes.data, None)

    def _download_2d(self, which, dtype):
        flat = self._dev.download(which, self.nrows * self.width, dtype)
        return np.asfortranarray(flat.reshape(self.width, self.nrows).T)

    col_idx = property(lambda s: s._get("col_idx", lambda: s._download_2d(_lib.ARR_COLS, np.int64)))
    values = property(lambda s: s._get("values", lambda: s._download_2d(_lib.ARR_VALS, np.float64)))

    @property
    def nnz(self) -> int:
        if self._dev is not None:
            return int(self._dev.info.nnz)
        return int(np.count_nonzero(self.col_idx != self.ncols)) if self.width else 0


class DiaMatrix(_Resident):
    """Stored diagonals: ``data[k, i]`` is the entry at (i, i + offsets[k])
    (formats.py:189-227)."""

    _tag = FormatTag.DIA

    def __init__(self, nrows, ncols, offsets, data):
        if nrows < 1 or ncols < 1:
            raise ValueError("matrix dimensions must be positive")
        self.nrows, self.ncols = int(nrows), int(ncols)
        o = _index_vector(offsets, "offsets")
        d = np.ascontiguousarray(data, dtype=np.float64)
        if d.shape != (o.size, self.nrows):
            raise ValueError("data must be len(offsets) x nrows")
        if o.size:
            if (np.diff(o) <= 0).any():
                raise ValueError("offsets must be strictly increasing")
            if o.min() <= -self.nrows or o.max() >= self.ncols:
                raise ValueError("offset out of range")
            if not np.isfinite(d).all():
                raise ValueError("data contains non-finite entries")
            i = np.arange(self.nrows)
            for k, off in enumerate(o.tolist()):
                out = (i + off < 0) | (i + off >= self.ncols)
                if (d[k, out] != 0.0).any():
                    raise ValueError("padding outside the matrix must be 0")
        self._ndiag = int(o.size)
        self._init_resident()
        self._host = {"offsets": _frozen(o), "data": _frozen(d)}

    @classmethod
    def _wrap(cls, dev: DeviceMatrix):
        self = cls.__new__(cls)
        self.nrows, self.ncols = int(dev.info.nrows), int(dev.info.ncols)
        self._ndiag = int(dev.info.ndiag)
        self._init_resident(dev)
        return self

    def _upload(self):
        return _new_handle(_lib.lib().svb_dia_create, self.nrows, self.ncols, self._ndiag,
                           self.offsets.ctypes.data, self.data.ctypes.data, None)

    offsets = property(lambda s: s._get("offsets", lambda: s._dev.download(
        _lib.ARR_OFFSETS, s._ndiag, np.int64)))
    data = property(lambda s: s._get("data", lambda: s._dev.download(
        _lib.ARR_DATA, s._ndiag * s.nrows, np.float64).reshape(s._ndiag, s.nrows)))

    @property
    def ndiag(self) -> int:
        return self._ndiag


class HybMatrix(_Resident):
    """ELL part holding up to ``split_width`` leading entries per row plus a
    COO spill (formats.py:230-260)."""

    _tag = FormatTag.HYB

    def __init__(self, ell_part: EllMatrix, coo_part: CooMatrix, split_width: int):
        if ell_part.nrows != coo_part.nrows or ell_part.ncols != coo_part.ncols:
            raise ValueError("ELL and COO parts must share dimensions")
        if ell_part.width != split_width:
            raise ValueError("ELL part width must equal split_width")
        stored = ell_part.col_idx != ell_part.ncols
        er, ek = np.nonzero(stored)
        flat_ell = er * ell_part.ncols + ell_part.col_idx[er, ek]
        flat_coo = coo_part.rows * coo_part.ncols + coo_part.cols
        if np.intersect1d(flat_ell, flat_coo).size:
            raise ValueError("a coordinate appears in both HYB parts")
        self.ell_part, self.coo_part, self.split_width = ell_part, coo_part, int(split_width)
        self._init_resident()

    @classmethod
    def _wrap(cls, dev: DeviceMatrix):
        self = cls.__new__(cls)
        self._init_resident(dev)
        self.split_width = int(dev.info.width)
        self._nrows, self._ncols = int(dev.info.nrows), int(dev.info.ncols)
        self._parts = None
        return self

    def _upload(self):
        return _new_handle(_lib.lib().svb_hyb_create, self.ell_part._device().handle,
                           self.coo_part._device().handle, None)

    def __getattr__(self, name):
        # device-born HYB: materialise the two parts on first access
        if name in ("ell_part", "coo_part"):
            parts = self.__dict__.get("_parts")
            if parts is None:
                parts = self._materialise_parts()
                self.__dict__["_parts"] = parts
                self.__dict__["ell_part"], self.__dict__["coo_part"] = parts
            return self.__dict__[name]
        raise AttributeError(name)

    def _materialise_parts(self):
        d = self._dev
        n, m, w = int(d.info.nrows), int(d.info.ncols), int(d.info.width)
        s = int(d.info.spill_nnz)
        ec = d.download(_lib.ARR_COLS, n * w, np.int64).reshape(w, n).T
        ev = d.download(_lib.ARR_VALS, n * w, np.float64).reshape(w, n).T
        ell = EllMatrix(n, m, w, ec, ev)
        coo = CooMatrix(n, m, d.download(_lib.ARR_ROWS, s, np.int64),
                        d.download(_lib.ARR_SPILL_COLS, s, np.int64),
                        d.download(_lib.ARR_SPILL_VALS, s, np.float64))
        return ell, coo

    @property
    def nrows(self) -> int:
        return self._nrows if "_nrows" in self.__dict__ else self.ell_part.nrows

    @property
    def ncols(self) -> int:
        return self._ncols if "_ncols" in self.__dict__ else self.ell_part.ncols

    @property
    def nnz(self) -> int:
        if self._dev is not None:
            return int(self._dev.info.nnz)
        return self.ell_part.nnz + self.coo_part.nnz


AnyMatrix = CooMatrix | CsrMatrix | EllMatrix | DiaMatrix | HybMatrix

_CLASS_OF = {FormatTag.COO: CooMatrix, FormatTag.CSR: CsrMatrix, FormatTag.ELL: EllMatrix,
             FormatTag.DIA: DiaMatrix, FormatTag.HYB: HybMatrix}
FORMAT_OF_TYPE = {cls: tag for tag, cls in _CLASS_OF.items()}


def format_of(m) -> FormatTag:
    try:
        return FORMAT_OF_TYPE[type(m)]
    except KeyError:
        raise TypeError(f"not a sparse matrix container: {type(m)!r}") from None


def convert(m, target: FormatTag, *, stream=None):
    """Convert ``m`` to ``target`` on the device (formats.py:302-320).

    Raises FormatInapplicableError for DIA above DIA_OFFSET_CAP diagonals
    and for ELL/HYB layouts beyond the device cell cap."""
    target = FormatTag(target)
    format_of(m)
    src = m._device()
    cap = max(ELL_MIN_CELLS, ELL_PAD_FACTOR * int(src.info.nnz))
    dev = _new_handle(_lib.lib().svb_convert, src.handle, _TAG_CODE[target], cap,
                      stream)
    return _CLASS_OF[target]._wrap(dev)


def to_coo(m) -> CooMatrix:
    """Any layout to coordinate form, as a fresh container (formats.py:281-299)."""
    return convert(m, FormatTag.COO)


def hyb_split_width(row_lengths) -> int:
    """Smallest width fully covering at least two thirds of the rows
    (formats.py:364-370).  Host helper over a length vector; the device
    conversion evaluates the same rule from a row-length histogram."""
    lens = np.asarray(row_lengths)
    if lens.size == 0:
        return 0
    need = (2 * lens.size + 2) // 3
    return int(np.partition(lens, need - 1)[need - 1])


def spmv_reference(m: CsrMatrix, x) -> np.ndarray:
    """y = A x accumulating each row in ascending column order from 0
    (formats.py:419-435), evaluated by the sequential-order device kernel."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (m.ncols,):
        raise ValueError(f"x must have length {m.ncols}, got {x.shape}")
    if not isinstance(m, CsrMatrix):
        raise TypeError("spmv_reference expects a CsrMatrix")
    from . import device
    return device.sequential_spmv_host(m, x)
