"""SpMV configuration space and the ``execute_spmv`` operator.

Drop-in for the reference ``spmvtune.kernels`` (kernels.py:1-312): the same
13-point (format, library, lane-width) space, token syntax, support table,
worker semantics and error messages.  Every configuration executes as a
hand-written sm_100a kernel (csrc/spmv.cu); the three "libraries" keep the
reference's distinct parallelisation strategies and summation orders:

* LibA — COO segmented reduction, CSR-vector with L lanes per row, ELL
  column sweep, DIA diagonal sweep, HYB (ELL + COO spill);
* LibB — COO scatter with fp64 atomics (nondeterministic, as in the
  reference) and CSR row-scalar;
* LibC — CSR merge-path chunks (``workers`` chunks) and column-strided ELL.

``x`` may be a numpy vector (host: H2D, kernel, D2H — the reference's
calling convention) or a device buffer (``DeviceVector``/torch CUDA tensor,
no copies).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .errors import UnsupportedConfigError
from .formats import FormatTag, format_of

LANE_WIDTHS = (2, 4, 8, 16, 32)

_WORKERS_ENV = "SPMVTUNE_WORKERS"
_workers_fixed: int | None = None


class Library(str, Enum):
    LIB_A = "LibA"
    LIB_B = "LibB"
    LIB_C = "LibC"


SUPPORT_TABLE = {  # kernels.py:43-47
    Library.LIB_A: frozenset(FormatTag),
    Library.LIB_B: frozenset({FormatTag.COO, FormatTag.CSR}),
    Library.LIB_C: frozenset({FormatTag.CSR, FormatTag.ELL}),
}

_LIB_CODE = {Library.LIB_A: _lib.LIBA, Library.LIB_B: _lib.LIBB, Library.LIB_C: _lib.LIBC}
_FMT_CODE = {FormatTag.COO: _lib.COO, FormatTag.CSR: _lib.CSR, FormatTag.ELL: _lib.ELL,
             FormatTag.DIA: _lib.DIA, FormatTag.HYB: _lib.HYB}


@dataclass(frozen=True)
class SpmvConfig:
    """A point of the configuration space (kernels.py:50-86)."""

    format: FormatTag
    library: Library
    lane_width: int | None = None

    def __post_init__(self):
        if self.format not in SUPPORT_TABLE[self.library]:
            raise UnsupportedConfigError(
                f"{self.library.value} does not implement {self.format.value}")
        if self.format is FormatTag.CSR and self.library is Library.LIB_A:
            if self.lane_width not in LANE_WIDTHS:
                raise UnsupportedConfigError(
                    f"lane_width must be one of {LANE_WIDTHS} for the lane-vectorized CSR "
                    f"kernel, got {self.lane_width!r}")
        elif self.lane_width is not None:
            raise UnsupportedConfigError("lane_width applies only to the LibA CSR kernel")

    def token(self) -> str:
        """``FMT/Lib`` or ``CSR/LibA/<lane>``."""
        head = f"{self.format.value}/{self.library.value}"
        return head if self.lane_width is None else f"{head}/{self.lane_width}"

    @classmethod
    def from_token(cls, token: str) -> "SpmvConfig":
        bits = token.split("/")
        if len(bits) not in (2, 3):
            raise UnsupportedConfigError(f"malformed config token {token!r}")
        lane = int(bits[2]) if len(bits) == 3 else None
        return cls(FormatTag(bits[0]), Library(bits[1]), lane)


DEFAULT_CONFIG = SpmvConfig(FormatTag.COO, Library.LIB_A)   # kernels.py:89
# The B200 solve starts on CSR-vector (BASELINE.json north star); API parity
# keeps DEFAULT_CONFIG, the backend default is selected explicitly.
GPU_DEFAULT_CONFIG = SpmvConfig(FormatTag.CSR, Library.LIB_A, 32)


def enumerate_configs() -> list[SpmvConfig]:
    """The 13 valid configurations in the reference's fixed order
    (kernels.py:92-108); the first is the default."""
    out = [DEFAULT_CONFIG]
    out += [SpmvConfig(FormatTag.CSR, Library.LIB_A, w) for w in LANE_WIDTHS]
    out += [SpmvConfig(FormatTag.ELL, Library.LIB_A), SpmvConfig(FormatTag.DIA, Library.LIB_A),
            SpmvConfig(FormatTag.HYB, Library.LIB_A), SpmvConfig(FormatTag.COO, Library.LIB_B),
            SpmvConfig(FormatTag.CSR, Library.LIB_B), SpmvConfig(FormatTag.CSR, Library.LIB_C),
            SpmvConfig(FormatTag.ELL, Library.LIB_C)]
    return out


def default_workers() -> int:
    """LibC chunk count, fixed per process; ``SPMVTUNE_WORKERS`` overrides
    (kernels.py:111-122)."""
    global _workers_fixed
    if _workers_fixed is None:
        env = os.environ.get(_WORKERS_ENV, "")
        _workers_fixed = int(env) if env else (os.cpu_count() or 1)
        if _workers_fixed < 1:
            raise ValueError(f"{_WORKERS_ENV} must be >= 1")
    return _workers_fixed


def _is_device_buffer(a) -> bool:
    if hasattr(a, "ptr") and hasattr(a, "n"):        # device.DeviceVector
        return True
    return getattr(a, "is_cuda", False)              # torch CUDA tensor


def _device_operand(a, name: str) -> tuple[int, str]:
    """(length, "float32"|"float64") of a device SpMV operand; raises
    ValueError for any other dtype, a non-contiguous tensor or a tensor on
    another device than the current one."""
    if hasattr(a, "n"):                                  # DeviceVector: flat by construction
        kind = np.dtype(a.dtype).name
        n = a.n
    else:
        kind = str(a.dtype).replace("torch.", "")
        if a.dim() != 1 or not a.is_contiguous():
            raise ValueError(f"{name} must be a contiguous 1-D device vector")
        dev = _lib.device_index()
        if a.device.index is not None and a.device.index != dev:
            raise ValueError(f"{name} lives on {a.device}, not the library's device cuda:{dev}")
        n = a.numel()
    if kind not in ("float32", "float64"):
        raise ValueError(f"{name} must be float32 or float64, got {kind}")
    return n, kind


def launch(cfg: SpmvConfig, m, x_ptr: int, y_ptr: int, *, workers: int, f32: bool = False,
           stream=None) -> None:
    """Enqueue y = A x on ``stream`` with raw device pointers (no checks
    beyond the C ABI's); the solver's per-iteration entry point."""
    _lib.check(_lib.lib().svb_spmv(m._device().handle, _FMT_CODE[cfg.format], _LIB_CODE[cfg.library],
                                   cfg.lane_width or 0, int(workers), _lib.F32 if f32 else _lib.F64,
                                   x_ptr, y_ptr, stream.handle if stream is not None else None))


def execute_spmv(cfg: SpmvConfig, m, x, *, workers: int | None = None, out=None, stream=None):
    """Run one SpMV under ``cfg`` (kernels.py:274-312).

    ``m`` must already be stored in ``cfg.format``.  With a numpy ``x`` the
    result is written into ``out`` (zero-filled semantics, returned by
    identity) or a fresh float64 vector.  With device buffers (``x`` a
    DeviceVector or CUDA tensor) the kernel is only enqueued; float32
    device buffers select the fp32 kernels."""
    if workers is None:
        workers = default_workers()
    if format_of(m) is not cfg.format:
        raise UnsupportedConfigError(
            f"matrix is stored as {format_of(m).value}, kernel expects {cfg.format.value}")
    if _is_device_buffer(x):
        n_x, kind_x = _device_operand(x, "x")
        if n_x != m.ncols:
            raise ValueError(f"x must have length {m.ncols}, got ({n_x},)")
        f32 = kind_x == "float32"
        if out is None:
            if hasattr(x, "n"):
                from .device import DeviceVector
                out = DeviceVector(m.nrows, np.float32 if f32 else np.float64)
            else:
                out = x.new_empty(m.nrows)
        else:
            # the kernel writes raw pointers: a short, mistyped or strided
            # out would be silent device-memory corruption
            if not _is_device_buffer(out):
                raise ValueError("out must be a device buffer when x is one")
            n_o, kind_o = _device_operand(out, "out")
            if n_o != m.nrows or kind_o != kind_x:
                raise ValueError(f"out must be a {kind_x} vector of length {m.nrows}, "
                                 f"got {kind_o} of length {n_o}")
        launch(cfg, m, _lib.ptr(x) if not hasattr(x, "n") else x.ptr,
               _lib.ptr(out) if not hasattr(out, "n") else out.ptr, workers=workers, f32=f32,
               stream=stream)
        return out
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (m.ncols,):
        raise ValueError(f"x must have length {m.ncols}, got {x.shape}")
    if out is None:
        out = np.zeros(m.nrows, dtype=np.float64)
    elif out.shape != (m.nrows,) or out.dtype != np.float64:
        raise ValueError("out must be a float64 vector of length nrows")
    if not out.flags.c_contiguous or not out.flags.writeable:
        raise ValueError("out must be a writeable contiguous float64 vector")
    _lib.check(_lib.lib().svb_spmv_host(m._device().handle, _FMT_CODE[cfg.format],
                                        _LIB_CODE[cfg.library], cfg.lane_width or 0, int(workers),
                                        x.ctypes.data, out.ctypes.data,
                                        stream.handle if stream is not None else None))
    return out
