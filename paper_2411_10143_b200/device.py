"""Thin host-side plumbing over the C ABI: streams, events, device vectors.

Nothing here computes; it only moves bytes and orders work.  Solver and
advisor work run on separate non-blocking CUDA streams (the advisor's at the
highest priority: its few short kernels are dispatched ahead of the solver's
queue instead of starving behind the persistent Arnoldi kernels) so the
paper's predict-while-solve overlap happens on the device, not just in host
threads.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib

_tls = threading.local()


class Stream:
    """Owned non-blocking CUDA stream (priority: +1 high, 0 normal, -1 low)."""

    def __init__(self, priority: int = 0):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().svb_stream_create(priority, ctypes.byref(h)))
        self.handle = h.value

    def sync(self):
        _lib.check(_lib.lib().svb_stream_sync(self.handle))

    def record(self) -> "Event":
        return Event(self)

    def wait(self, ev: "Event"):
        _lib.check(_lib.lib().svb_stream_wait_event(self.handle, ev.handle))

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.load().svb_stream_sync(h)
                _lib.load().svb_stream_destroy(h)
            except Exception:
                pass


class Event:
    def __init__(self, stream: Stream | None):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().svb_event_record(stream.handle if stream else None, ctypes.byref(h)))
        self.handle = h.value

    def sync(self):
        _lib.check(_lib.lib().svb_event_sync(self.handle))

    def done(self) -> bool:
        st = _lib.lib().svb_event_query(self.handle)
        if st == _lib.OK:
            return True
        if st == _lib.INVALID:
            return False
        _lib.check(st)
        return False

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.load().svb_event_destroy(h)
            except Exception:
                pass


def thread_stream(priority: int = 0) -> Stream:
    """A per-thread stream (created on first use)."""
    key = f"s{priority}"
    s = getattr(_tls, key, None)
    if s is None:
        s = Stream(priority)
        setattr(_tls, key, s)
    return s


_shared = {}
_shared_lock = threading.Lock()


def shared_stream(priority: int) -> Stream:
    """A process-wide stream (created once): advisor threads are short-lived,
    and creating/destroying a CUDA stream per solve costs milliseconds."""
    s = _shared.get(priority)
    if s is None:
        with _shared_lock:
            s = _shared.get(priority)
            if s is None:
                s = _shared[priority] = Stream(priority)
    return s


class DeviceVector:
    """A device buffer of ``n`` elements (float64 by default)."""

    def __init__(self, n: int, dtype=np.float64):
        self.n = int(n)
        self.dtype = np.dtype(dtype)
        p = ctypes.c_void_p()
        _lib.check(_lib.lib().svb_malloc(self.nbytes, ctypes.byref(p)))
        self.ptr = p.value or 0

    @property
    def nbytes(self) -> int:
        return self.n * self.dtype.itemsize

    @classmethod
    def from_numpy(cls, a: np.ndarray, stream: Stream | None = None) -> "DeviceVector":
        a = np.ascontiguousarray(a)
        v = cls(a.size, a.dtype)
        copy_host(v.ptr, a.ctypes.data, v.nbytes, True, stream)
        if stream is None:
            _lib.check(_lib.lib().svb_stream_sync(None))
        else:
            stream.sync()
        return v

    def to_numpy(self, stream: Stream | None = None) -> np.ndarray:
        out = np.empty(self.n, self.dtype)
        copy_host(out.ctypes.data, self.ptr, self.nbytes, False, stream)
        _lib.check(_lib.lib().svb_stream_sync(stream.handle if stream else None))
        return out

    def __del__(self):
        p, self.ptr = getattr(self, "ptr", 0), 0
        if p:
            try:
                _lib.load().svb_free(p)
            except Exception:
                pass


def copy(dst: int, src: int, nbytes: int, stream: Stream | None = None) -> None:
    if int(nbytes) == 0:         # zero-length vectors (a rank without rows) have no pointer
        return
    _lib.check(_lib.lib().svb_copy(dst, src, int(nbytes), stream.handle if stream else None))


def copy_host(dst: int, src: int, nbytes: int, to_device: bool, stream: Stream | None = None) -> None:
    """Host (numpy) buffer <-> device, blocking: downloads of 12 MB and more
    into pageable buffers go through the library's multi-threaded pinned
    staging (svb_copy_host); everything else copies directly."""
    if int(nbytes) == 0:
        return
    _lib.check(_lib.lib().svb_copy_host(dst, src, int(nbytes), 1 if to_device else 0,
                                        stream.handle if stream else None))


def memset(dst: int, value: int, nbytes: int, stream: Stream | None = None) -> None:
    if int(nbytes) == 0:
        return
    _lib.check(_lib.lib().svb_memset(dst, value, int(nbytes), stream.handle if stream else None))


def sequential_spmv_host(m, x: np.ndarray) -> np.ndarray:
    """spmv_reference on the device: H2D x, sequential-order kernel, D2H y."""
    s = thread_stream()
    xd = DeviceVector.from_numpy(x, s)
    yd = DeviceVector(m.nrows)
    _lib.check(_lib.lib().svb_spmv_sequential(m._device().handle, xd.ptr, yd.ptr, s.handle))
    return yd.to_numpy(s)


def device_info() -> dict:
    sms = ctypes.c_int32()
    free = ctypes.c_int64()
    total = ctypes.c_int64()
    _lib.check(_lib.lib().svb_device_info(ctypes.byref(sms), ctypes.byref(free), ctypes.byref(total)))
    res, used = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().svb_pool_info(ctypes.byref(res), ctypes.byref(used)))
    return {"sm_count": sms.value, "free_bytes": free.value, "total_bytes": total.value,
            "pool_reserved_bytes": res.value, "pool_used_bytes": used.value}
