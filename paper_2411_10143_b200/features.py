"""Structural features of a CSR matrix, extracted on the B200.

Drop-in for the reference ``spmvtune.features`` (features.py:1-156).  The
device (csrc/features.cu) computes the seven exact integer aggregates in one
fused pass plus a popcount; the fifteen float features are then evaluated
here with the reference's own expressions and operation order
(features.py:103-110, 147-150), which makes the vector bit-identical to the
CPU path.

Cancellation keeps the reference contract (features.py:60-65, 89-91): a
flag raised before the call returns ``None`` without reading ``row_ptr`` or
``col_idx``; a flag raised while the pass runs is forwarded to the device
(a host-mapped word the kernel polls once per 256-row tile), which then
stops reading, and the call returns ``None``.  The traversal counters report
the row_ptr and col_idx elements the device pass actually read.
"""
from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .formats import CsrMatrix

FEATURE_NAMES = ("nrows", "ncols", "nnz", "density", "mean", "sd", "cov", "max", "min",
                 "maxavg", "distavg", "clusteravg", "fill", "ndiag", "diagfill")

CANCEL_CHECK_ROWS = 4096


@dataclass
class FeatureVector:
    nrows: int
    ncols: int
    nnz: int
    density: float
    mean: float
    sd: float
    cov: float
    max: float
    min: float
    maxavg: float
    distavg: float
    clusteravg: float
    fill: float
    ndiag: float
    diagfill: float

    def to_array(self) -> np.ndarray:
        return np.array([getattr(self, k) for k in FEATURE_NAMES], dtype=np.float64)

    @classmethod
    def from_array(cls, a) -> "FeatureVector":
        a = np.asarray(a, dtype=np.float64)
        if a.shape != (len(FEATURE_NAMES),):
            raise ValueError(f"expected {len(FEATURE_NAMES)} features, got shape {a.shape}")
        kw = dict(zip(FEATURE_NAMES, a))
        for k in ("nrows", "ncols", "nnz"):
            kw[k] = int(kw[k])
        return cls(**kw)


@dataclass
class TraversalCounter:
    """Array elements consumed by an extraction (features.py:60-65)."""

    row_ptr_reads: int = 0
    col_idx_reads: int = 0


def device_aggregates(m: CsrMatrix, stream=None) -> tuple[int, int, int, int, int, int, int]:
    """(sum r, sum r^2, max r, min r, sum span, sum longest run, ndiag)."""
    agg = (ctypes.c_int64 * 7)()
    _lib.check(_lib.lib().svb_features(m._device().handle, agg,
                                       stream.handle if stream is not None else None))
    return tuple(int(v) for v in agg)


def features_from_aggregates(nrows: int, ncols: int, nnz: int, agg) -> FeatureVector:
    """The reference's float formulas over exact integers (Python ints, true
    division, numpy sqrt) — evaluated in the same order as features.py."""
    sum_r, sum_r2, max_r, min_r, span_sum, run_sum, ndiag = agg
    density = nnz / (nrows * ncols)
    mean = nnz / nrows
    sd = float(np.sqrt(max(sum_r2 / nrows - mean * mean, 0.0)))
    cov = sd / mean if mean > 0 else 0.0
    maxavg = max_r - mean
    fill = nrows * max_r / nnz if nnz > 0 else 0.0
    distavg = span_sum / nrows
    clusteravg = run_sum / nrows
    diagfill = nrows * ndiag / nnz if nnz > 0 else 0.0
    return FeatureVector(nrows=nrows, ncols=ncols, nnz=nnz, density=density, mean=mean, sd=sd,
                         cov=cov, max=float(max_r), min=float(min_r or 0), maxavg=maxavg,
                         distavg=distavg, clusteravg=clusteravg, fill=fill, ndiag=float(ndiag),
                         diagfill=diagfill)


class CancelEvent(threading.Event):
    """A threading.Event that also runs registered hooks when it is set (in
    the setting thread).  The solver's convergence flag is one: a feature
    pass blocked in native code (svb_features_wait, GIL released) is
    cancelled by a hook instead of a Python thread polling the event, whose
    wake-ups every 50 us contend for the GIL with the solver loop."""

    def __init__(self):
        super().__init__()
        self._hooks: list = []
        self._hooks_lock = threading.Lock()

    def add_hook(self, fn) -> None:
        with self._hooks_lock:
            self._hooks.append(fn)

    def remove_hook(self, fn) -> None:
        with self._hooks_lock:
            if fn in self._hooks:
                self._hooks.remove(fn)

    def set(self) -> None:
        super().set()
        with self._hooks_lock:
            hooks = list(self._hooks)
        for fn in hooks:
            fn()


def extract_features(m: CsrMatrix, cancel: threading.Event | None = None, *,
                     counter: TraversalCounter | None = None,
                     row_chunk: int = CANCEL_CHECK_ROWS, stream=None) -> FeatureVector | None:
    """Feature vector of ``m`` or ``None`` when ``cancel`` is (or becomes) set.

    The device pass runs as a job (svb_features_start); while it runs this
    thread polls ``cancel`` and forwards a raised flag to the kernel, which
    stops at its next 256-row tile — the device analogue of the reference's
    check every ``row_chunk`` rows (accepted for API parity)."""
    if cancel is not None and cancel.is_set():
        return None
    if not isinstance(m, CsrMatrix):
        raise TypeError("extract_features expects a CsrMatrix")
    L = _lib.lib()
    job = ctypes.c_void_p()
    _lib.check(L.svb_features_start(m._device().handle, 0, stream.handle if stream is not None else None,
                                    ctypes.byref(job)))
    agg = (ctypes.c_int64 * 7)()
    cnt = (ctypes.c_int64 * 2)()
    was = ctypes.c_int32(0)
    try:
        if isinstance(cancel, CancelEvent):
            # block in native code; a set() from the solver thread forwards
            # the cancel through the hook (serialised with its retirement)
            live, lock = [True], threading.Lock()

            def hook():
                with lock:
                    if live[0]:
                        _lib.check(L.svb_features_cancel(job))
            cancel.add_hook(hook)
            try:
                if cancel.is_set():
                    hook()
                _lib.check(L.svb_features_wait(job))
            finally:
                with lock:
                    live[0] = False
                cancel.remove_hook(hook)
        elif cancel is not None:
            done = ctypes.c_int32(0)
            forwarded = False
            while True:
                _lib.check(L.svb_features_query(job, ctypes.byref(done)))
                if done.value:
                    break
                if forwarded:
                    time.sleep(20e-6)
                elif cancel.wait(50e-6):
                    _lib.check(L.svb_features_cancel(job))
                    forwarded = True
    finally:
        _lib.check(L.svb_features_finish(job, agg, cnt, ctypes.byref(was)))
    if counter is not None:
        counter.row_ptr_reads += int(cnt[0])
        counter.col_idx_reads += int(cnt[1])
    if was.value or (cancel is not None and cancel.is_set()):
        return None
    return features_from_aggregates(m.nrows, m.ncols, m.nnz, tuple(int(v) for v in agg))
