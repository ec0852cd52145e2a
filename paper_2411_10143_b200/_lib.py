"""ctypes binding of libspmvtune_b200.so (the C ABI in include/spmvtune_b200.h).

Loading is lazy but loud: every product entry point goes through ``lib()``,
which raises ImportError if the in-tree library was not built.  There is no
CPU fallback anywhere in the package.  Non-zero statuses map onto the
reference's exception hierarchy (errors.py:4-29) via ``check``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import (FormatInapplicableError, MatrixMarketError, SolverNumericalError,
                     UnsupportedConfigError)

LIB_PATH = Path(__file__).resolve().parent / "libspmvtune_b200.so"
if os.environ.get("SPMVTUNE_LIB_VARIANT"):        # A/B experiments on kernel variants
    LIB_PATH = LIB_PATH.with_name(f"libspmvtune_b200_{os.environ['SPMVTUNE_LIB_VARIANT']}.so")

OK, UNSUPPORTED, INAPPLICABLE, DIM_MISMATCH, NONFINITE, OOM, CUDA, INVALID, FORMAT_ERROR = range(9)
COO, CSR, ELL, DIA, HYB = range(5)
LIBA, LIBB, LIBC = range(3)
F64, F32 = 0, 1
ARR_ROW_PTR, ARR_ROWS, ARR_COLS, ARR_VALS, ARR_OFFSETS, ARR_DATA, ARR_SPILL_COLS, ARR_SPILL_VALS = range(8)

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_PI64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)
_PP = C.POINTER(C.c_void_p)


class MatrixInfo(C.Structure):
    _fields_ = [("format", C.c_int32), ("ptr64", C.c_int32), ("nrows", C.c_int64),
                ("ncols", C.c_int64), ("nnz", C.c_int64), ("width", C.c_int64),
                ("ndiag", C.c_int64), ("spill_nnz", C.c_int64), ("device_bytes", C.c_int64)]


class KrylovStatus(C.Structure):
    _fields_ = [("beta", C.c_double), ("hnext", C.c_double), ("estimate", C.c_double),
                ("hjj", C.c_double), ("pq", C.c_double), ("nonfinite", C.c_int32),
                ("done", C.c_int32), ("count", C.c_int64)]


class SvbConfig(C.Structure):
    _fields_ = [("format", C.c_int32), ("library", C.c_int32), ("lane", C.c_int32),
                ("workers", C.c_int32)]


class SolveParams(C.Structure):
    _fields_ = [("restart_m", C.c_int32), ("max_iters", C.c_int32), ("tol", C.c_double)]


class Swap(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("config", SvbConfig), ("prep_seconds", C.c_double)]


class SolveReportC(C.Structure):
    _fields_ = [("converged", C.c_int32), ("stagnated", C.c_int32), ("iterations", C.c_int32),
                ("history_len", C.c_int32), ("nswaps", C.c_int32), ("final_residual", C.c_double)]


# name -> argtypes (all functions return int status unless listed in _RESTYPE)
_SIGS = {
    "svb_last_error": [],
    "svb_abi_version": [],
    "svb_launch_count": [_PI64],
    "svb_init": [C.c_int],
    "svb_stream_sync": [_P],
    "svb_stream_create": [C.c_int, _PP],
    "svb_stream_destroy": [_P],
    "svb_event_record": [_P, _PP],
    "svb_event_query": [_P],
    "svb_stream_wait_event": [_P, _P],
    "svb_event_destroy": [_P],
    "svb_malloc": [_I64, _PP],
    "svb_free": [_P],
    "svb_host_alloc": [_I64, _PP],
    "svb_host_free": [_P],
    "svb_copy": [_P, _P, _I64, _P],
    "svb_copy_host": [_P, _P, _I64, _I32, _P],
    "svb_memset": [_P, C.c_int, _I64, _P],
    "svb_device_info": [C.POINTER(C.c_int32), _PI64, _PI64],
    "svb_pool_info": [_PI64, _PI64],
    "svb_coo_create": [_I64, _I64, _I64, _P, _P, _P, _P, _PP],
    "svb_csr_create": [_I64, _I64, _I64, _P, _P, _P, _P, _PP],
    "svb_ell_create": [_I64, _I64, _I64, _P, _P, _P, _PP],
    "svb_dia_create": [_I64, _I64, _I64, _P, _P, _P, _PP],
    "svb_hyb_create": [_P, _P, _P, _PP],
    "svb_matrix_destroy": [_P],
    "svb_matrix_info_get": [_P, C.POINTER(MatrixInfo)],
    "svb_matrix_download": [_P, C.c_int, _P, _P],
    "svb_csr_stencil": [C.c_int, _PI64, C.c_int, C.POINTER(C.c_int32), _PD, _P, _PP],
    "svb_fill": [_P, C.c_int64, C.c_double, _P],
    "svb_mm_open": [C.c_char_p, _PI64, C.POINTER(C.c_int32), _PP],
    "svb_mm_parse": [_P, _P, _P, _P, C.c_int32],
    "svb_mm_close": [_P],
    "svb_coo_from_triplets": [C.c_int64, C.c_int64, C.c_int64, _P, _P, _P, C.c_int32, _P, _PP],
    "svb_event_sync": [_P],
    "svb_dcg_rupdate": [_P, _P, _I32, _I32, _I32, _I32, _P, _P, _P],
    "svb_peer_create": [C.c_int, C.c_int, C.POINTER(C.c_void_p)],
    "svb_peer_destroy": [_P],
    "svb_peer_mailbox": [_P, C.POINTER(C.c_void_p)],
    "svb_peer_set_mailbox": [_P, C.c_int, _P],
    "svb_peer_alloc": [C.c_int64, C.POINTER(C.c_void_p)],
    "svb_peer_free": [_P],
    "svb_peer_ipc_handle": [_P, _P],
    "svb_peer_ipc_open": [_P, C.POINTER(C.c_void_p)],
    "svb_peer_ipc_close": [_P],
    "svb_peer_error": [_P, C.POINTER(C.c_int)],
    "svb_peer_allreduce": [_P, _P, C.c_int, _P],
    "svb_peer_wait_halo": [_P, _P, C.c_int, _P],
    "svb_dcg_xp_push": [_P, C.c_int64, _P, _I32, _I32, _I32, _P, _P, _P, C.c_int, _P, _P, _P, _P, _P],
    "svb_dcg_xp": [_P, _P, _I32, _I32, _I32, _P, _P, _P, _P],
    "svb_cg_step_batched_dia": [_P, _P, C.c_double, _P],
    "svb_krylov_mark": [_P, _P],
    "svb_graph_begin": [_P],
    "svb_graph_end": [_P, _PP],
    "svb_graph_launch": [_P, _P],
    "svb_graph_destroy": [_P],
    "svb_csr_row_slice": [_P, C.c_int64, C.c_int64, _P, _PP],
    "svb_csr_create_slab": [_I64, _I64, _I64, _I64, _P, _P, _I32, _P, _P, _PI64, _PP],
    "svb_csr_export": [_P, _I64, _P, _P, _P, _P],
    "svb_diag_offsets": [_P, _I64, _PI64, _I64, _PI64, _P],
    "svb_mailbox_create": [_PP],
    "svb_mailbox_destroy": [_P],
    "svb_mailbox_publish": [_P, _P, SvbConfig, _P, C.c_double],
    "svb_mailbox_finished": [_P, C.POINTER(C.c_int32)],
    "svb_gmres_run": [_P, SvbConfig, _P, _P, C.POINTER(SolveParams), _P, _P, _PD, C.POINTER(Swap),
                      C.c_int32, C.POINTER(SolveReportC)],
    "svb_cg_run": [_P, SvbConfig, _P, _P, C.POINTER(SolveParams), _P, _P, _PD, C.POINTER(Swap),
                   C.c_int32, C.POINTER(SolveReportC)],
    "svb_csr_stencil_rows": [C.c_int, _PI64, C.c_int, C.POINTER(C.c_int32), _PD, C.c_int64, C.c_int64,
                             C.c_int64, C.c_int64, _P, _PP],
    "svb_convert": [_P, C.c_int, _I64, _P, _PP],
    "svb_hyb_split_width": [_P, _P, _PI64],
    "svb_spmv": [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P],
    "svb_spmv_host": [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P],
    "svb_spmv_sequential": [_P, _P, _P, _P],
    "svb_features": [_P, _PI64, _P],
    "svb_features_start": [_P, C.c_int, _P, _PP],
    "svb_features_cancel": [_P],
    "svb_features_query": [_P, C.POINTER(C.c_int32)],
    "svb_features_wait": [_P],
    "svb_features_finish": [_P, _PI64, _PI64, C.POINTER(C.c_int32)],
    "svb_krylov_create": [_I64, _I32, _PP],
    "svb_krylov_destroy": [_P],
    "svb_krylov_vec": [_P, C.c_int, _PP],
    "svb_krylov_status_get": [_P, _P, C.POINTER(KrylovStatus)],
    "svb_krylov_bnorm": [_P, _P],
    "svb_krylov_residual": [_P, _P],
    "svb_gmres_restart": [_P, _P],
    "svb_gmres_arnoldi": [_P, _I32, _D, _P],
    "svb_gmres_normalize": [_P, _I32, _P],
    "svb_gmres_update_x": [_P, _I32, _P],
    "svb_cg_restart": [_P, _P],
    "svb_cg_step": [_P, _D, _P],
    "svb_cg_batch_reset": [_P, _D, _I64, _P],
    "svb_cg_batch_resume": [_P, _P],
    "svb_cg_step_batched": [_P, _D, _P],
    "svb_cg_history": [_P, _I64, _I64, _PD, _P],
    "svb_dot": [_P, _P, _I64, _PD, _P],
    "svb_vecops_create": [_I64, _PP],
    "svb_vecops_destroy": [_P],
    "svb_vec_dot": [_P, _P, _P, _P, _P],
    "svb_vec_axpy_dot": [_P, _P, _D, _P, _P, _P, _P, _P],
    "svb_vec_axpby": [_P, _D, _P, _D, _P, _P],
    "svb_vec_scale": [_P, _P, _D, _P],
    "svb_vec_spmv_dot": [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, _I32, _P],
    "svb_vec_gs": [_P, _I32, _P, _I64, _I32, _P, _P, _P, _P, _P, _P],
    "svb_vec_gs_hn": [_P, _I32, _P, _P, _P],
    "svb_forest_create": [_I32, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _PP],
    "svb_forest_destroy": [_P],
    "svb_forest_predict": [_P, _P, _P, _P],
}
_RESTYPE = {"svb_last_error": C.c_char_p}

_lock = threading.Lock()
_lib = None
_initialised = False


def exported_symbols():
    """Names the header declares (checked against the .so by the CPU tests)."""
    return sorted(_SIGS)


def load():
    """dlopen the library and bind signatures (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH.name} is not built; run `python -m paper_2411_10143_b200.build` "
                    "(this package has no CPU fallback)")
            lib_ = C.CDLL(str(LIB_PATH))
            for name, args in _SIGS.items():
                fn = getattr(lib_, name)
                fn.argtypes = args
                fn.restype = _RESTYPE.get(name, C.c_int)
            _lib = lib_
    return _lib


def device_index() -> int:
    """The CUDA device this process's library calls run on (SPMVTUNE_DEVICE,
    else LOCAL_RANK, else 0)."""
    if os.environ.get("SPMVTUNE_DEVICE") is not None:
        return int(os.environ["SPMVTUNE_DEVICE"])
    return int(os.environ.get("LOCAL_RANK", "0"))


def lib():
    """The library, with the CUDA device selected for the calling process."""
    global _initialised
    L = load()
    if not _initialised:
        with _lock:
            if not _initialised:
                check(L.svb_init(device_index()))
                _initialised = True
    return L


def launch_count() -> int:
    n = C.c_int64()
    load().svb_launch_count(C.byref(n))
    return n.value


def last_error() -> str:
    raw = load().svb_last_error()
    return raw.decode("utf-8", "replace") if raw else ""


_EXC = {UNSUPPORTED: UnsupportedConfigError, INAPPLICABLE: FormatInapplicableError,
        DIM_MISMATCH: ValueError, NONFINITE: SolverNumericalError, OOM: MemoryError,
        CUDA: RuntimeError, INVALID: ValueError, FORMAT_ERROR: MatrixMarketError}


def check(status: int) -> None:
    if status != OK:
        raise _EXC.get(status, RuntimeError)(last_error() or f"spmvtune_b200 status {status}")


def ptr(a) -> int:
    """Raw address of a numpy array / torch tensor / int."""
    if a is None:
        return 0
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return int(a.data_ptr())
    return int(a.ctypes.data)
