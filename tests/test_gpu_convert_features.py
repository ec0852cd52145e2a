"""GPU parity: device conversions and feature extraction are bit-exact with
the reference (golden fixtures) and the oracle."""
import threading
import time

import numpy as np
import pytest

import oracle as O
from golden_io import case, case_names

import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G
from paper_2411_10143_b200.features import TraversalCounter

pytestmark = pytest.mark.gpu


def coo_of(c):
    return P.CooMatrix(int(c["nrows"]), int(c["ncols"]), c["coo_rows"], c["coo_cols"], c["coo_vals"])


@pytest.mark.parametrize("name", case_names())
def test_conversions_bit_exact(name):
    c = case(name)
    coo = coo_of(c)
    csr = P.convert(coo, P.FormatTag.CSR)
    assert np.array_equal(csr.row_ptr, c["csr_ptr"])
    assert np.array_equal(csr.col_idx, c["coo_cols"])
    assert np.array_equal(csr.values, c["coo_vals"])
    for src in (coo, csr):   # COO hub and CSR-direct paths
        ell = P.convert(src, P.FormatTag.ELL)
        assert ell.width == int(c["ell_width"])
        assert np.array_equal(ell.col_idx.T, c["ell_cols"])
        assert np.array_equal(ell.values.T, c["ell_vals"])
        hyb = P.convert(src, P.FormatTag.HYB)
        assert hyb.split_width == int(c["hyb_width"])
        assert np.array_equal(hyb.ell_part.col_idx.T, c["hyb_ell_cols"])
        assert np.array_equal(hyb.ell_part.values.T, c["hyb_ell_vals"])
        assert np.array_equal(hyb.coo_part.rows, c["hyb_spill_rows"])
        assert np.array_equal(hyb.coo_part.cols, c["hyb_spill_cols"])
        assert np.array_equal(hyb.coo_part.values, c["hyb_spill_vals"])
        if int(c["dia_ok"]):
            dia = P.convert(src, P.FormatTag.DIA)
            assert np.array_equal(dia.offsets, c["dia_offsets"])
            assert np.array_equal(dia.data, c["dia_data"])
        else:
            with pytest.raises(P.FormatInapplicableError, match="inapplicable"):
                P.convert(src, P.FormatTag.DIA)
    # round trips back through COO (to_coo of every layout)
    for fmt in (P.FormatTag.CSR, P.FormatTag.ELL, P.FormatTag.HYB, P.FormatTag.COO):
        back = P.to_coo(P.convert(coo, fmt))
        assert np.array_equal(back.rows, c["coo_rows"]), fmt
        assert np.array_equal(back.cols, c["coo_cols"]), fmt
        assert np.array_equal(back.values, c["coo_vals"]), fmt
    if int(c["dia_ok"]):
        back = P.to_coo(P.convert(coo, P.FormatTag.DIA))
        keep = c["coo_vals"] != 0.0
        assert np.array_equal(back.rows, c["coo_rows"][keep])
        assert np.array_equal(back.cols, c["coo_cols"][keep])


def test_host_built_containers_upload_and_convert():
    c = case("banded")
    coo = O.OCoo(int(c["nrows"]), int(c["ncols"]), c["coo_rows"], c["coo_cols"], c["coo_vals"])
    ell, dia, hyb = O.coo_to_ell(coo), O.coo_to_dia(coo), O.coo_to_hyb(coo)
    mats = [P.EllMatrix(ell.nrows, ell.ncols, ell.width, ell.cols, ell.vals),
            P.DiaMatrix(dia.nrows, dia.ncols, dia.offsets, dia.data),
            P.HybMatrix(P.EllMatrix(coo.nrows, coo.ncols, hyb.width, hyb.ell.cols, hyb.ell.vals),
                        P.CooMatrix(coo.nrows, coo.ncols, hyb.spill.rows, hyb.spill.cols,
                                    hyb.spill.vals), hyb.width)]
    for m in mats:
        csr = P.convert(m, P.FormatTag.CSR)
        assert np.array_equal(csr.row_ptr, c["csr_ptr"])
        assert np.array_equal(csr.col_idx, c["coo_cols"])
        assert np.array_equal(csr.values, c["coo_vals"])


@pytest.mark.parametrize("name", case_names())
def test_features_bit_exact(name):
    c = case(name)
    csr = P.convert(coo_of(c), P.FormatTag.CSR)
    fv = P.extract_features(csr)
    assert fv.to_array().tolist() == c["features"].tolist()


def test_features_large_against_oracle():
    for n, m, ptr, cols, vals in (G.powerlaw_spd(200000, seed=4), G.convdiff9(700),
                                  G.laplace27(40)):
        fv = P.extract_features(P.CsrMatrix(n, m, ptr, cols, vals))
        assert fv.to_array().tolist() == O.features(O.OCsr(n, m, ptr, cols, vals))


def test_features_extra_long_rows_against_oracle():
    """Rows longer than FEAT_XL (2048) are walked by a whole CTA in eight
    parts joined left to right (k_features_xl): runs that cross part
    boundaries, rows that are one run, alternating gaps, a run ending exactly
    at a part edge — the aggregates must equal the sequential recurrence."""
    rng = np.random.default_rng(3)
    ncols = 400_000
    rows = []
    rows.append(np.arange(1000, 1000 + 20_000))                       # one run
    r = np.arange(5000, 5000 + 30_000)
    rows.append(r[np.arange(r.size) % 7 != 3])                        # gaps every 7
    rows.append(np.arange(0, 2 * 9000, 2))                            # no two consecutive
    a = np.arange(100, 100 + 8 * 1000)                                # breaks at part edges
    rows.append(np.concatenate([a[:4000], a[4000:] + 50]))
    rows.append(np.sort(rng.choice(ncols, size=5000, replace=False)))
    blk = np.arange(200_000, 200_000 + 12_345)                        # long run inside random
    rows.append(np.unique(np.concatenate([blk, rng.choice(ncols, size=3000, replace=False)])))
    n = 3000
    body = [np.sort(rng.choice(ncols, size=int(rng.integers(1, 40)), replace=False)) for _ in range(n - len(rows))]
    allrows = body[:1000] + rows + body[1000:]
    ptr = np.zeros(n + 1, np.int64)
    ptr[1:] = np.cumsum([x.size for x in allrows])
    cols = np.concatenate(allrows).astype(np.int64)
    vals = np.ones(cols.size)
    fv = P.extract_features(P.CsrMatrix(n, ncols, ptr, cols, vals))
    assert fv.to_array().tolist() == O.features(O.OCsr(n, ncols, ptr, cols, vals))


def test_feature_cancellation_and_counters():
    n, m, ptr, cols, vals = G.poisson2d(40)
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    ev = threading.Event()
    ev.set()
    cnt = TraversalCounter()
    assert P.extract_features(csr, ev, counter=cnt) is None
    assert cnt.col_idx_reads == 0 and cnt.row_ptr_reads == 0
    cnt = TraversalCounter()
    assert P.extract_features(csr, counter=cnt, row_chunk=64) is not None
    assert cnt.col_idx_reads == csr.nnz
    assert cnt.row_ptr_reads <= 2 * (csr.nrows + 1) + 2 * (csr.nrows // 64 + 1)

    cancel = threading.Event()

    class Tripping(TraversalCounter):
        def __setattr__(self, k, v):
            super().__setattr__(k, v)
            if k == "col_idx_reads" and v > 0:
                cancel.set()

    assert P.extract_features(csr, cancel, counter=Tripping(), row_chunk=16) is None


def test_device_cancel_flag_stops_the_pass():
    """The cancel flag is device-visible: raised after the job is enqueued but
    before its kernel runs (the stream is held by a spin kernel), the pass
    reads no row_ptr/col_idx element and reports the cancellation; the next
    uncancelled pass on the same handle is complete and exact."""
    import ctypes
    torch = pytest.importorskip("torch")
    from paper_2411_10143_b200 import _lib, device
    n, m, ptr, cols, vals = G.convdiff9(300)
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    L = _lib.lib()
    s = device.thread_stream()
    h = csr._device().handle
    with torch.cuda.stream(torch.cuda.ExternalStream(s.handle)):
        torch.cuda._sleep(20_000_000)        # hold the stream ~10 ms
    job = ctypes.c_void_p()
    _lib.check(L.svb_features_start(h, 0, s.handle, ctypes.byref(job)))
    _lib.check(L.svb_features_cancel(job))
    agg, cnt, was = (ctypes.c_int64 * 7)(), (ctypes.c_int64 * 2)(), ctypes.c_int32(0)
    _lib.check(L.svb_features_finish(job, agg, cnt, ctypes.byref(was)))
    assert was.value == 1 and cnt[0] == 0 and cnt[1] == 0
    ctr = TraversalCounter()
    fv = P.extract_features(csr, threading.Event(), counter=ctr)
    assert fv.to_array().tolist() == O.features(O.OCsr(n, m, ptr, cols, vals))
    assert ctr.col_idx_reads == csr.nnz
    dia = P.convert(csr, P.FormatTag.DIA)      # from the offsets the pass left on the handle
    want = O.convert(O.OCsr(n, m, ptr, cols, vals), "DIA")
    assert np.array_equal(dia.offsets, want.offsets) and np.array_equal(dia.data, want.data)


def test_hooked_cancel_event_stops_a_blocked_pass():
    """extract_features with the solver's CancelEvent blocks in native code
    (svb_features_wait); set() from another thread cancels the running pass
    through the hook, the call returns None, and the handle's next pass is
    exact (the job was re-armed and recycled)."""
    torch = pytest.importorskip("torch")
    from paper_2411_10143_b200 import device
    from paper_2411_10143_b200.features import CancelEvent
    n, m, ptr, cols, vals = G.convdiff9(300)
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    s = device.thread_stream()
    csr._device()
    for delay in (0.0, 0.005):
        with torch.cuda.stream(torch.cuda.ExternalStream(s.handle)):
            torch.cuda._sleep(40_000_000)     # hold the stream ~20 ms
        ev, box, ctr = CancelEvent(), {}, TraversalCounter()
        th = threading.Thread(target=lambda: box.setdefault("fv", P.extract_features(csr, ev, counter=ctr,
                                                                                      stream=s)))
        th.start()
        time.sleep(delay)
        ev.set()
        th.join(timeout=30)
        assert not th.is_alive() and box["fv"] is None
        assert ctr.col_idx_reads < csr.nnz
        assert not ev._hooks                  # the hook was retired
    fv = P.extract_features(csr, CancelEvent(), stream=s)
    assert fv.to_array().tolist() == O.features(O.OCsr(n, m, ptr, cols, vals))


def test_device_stencil_generator_matches_host():
    for dims, gen in (((30, 30), G.poisson2d(30)), ((25, 25), G.convdiff9(25)),
                      ((9, 9, 9), G.laplace27(9))):
        n, _, ptr, cols, vals = gen
        offs, w = [], []
        if len(dims) == 2 and vals.max() == 4.0:
            offs, w = [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)], [4.0, -1, -1, -1, -1]
        elif len(dims) == 2:
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    offs.append((dy, dx))
                    w.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
        else:
            for dz in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        offs.append((dz, dy, dx))
                        w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
        dev = P.CsrMatrix.stencil(dims, offs, w)
        assert dev.nnz == cols.size
        assert np.array_equal(dev.row_ptr, ptr)
        assert np.array_equal(dev.col_idx, cols)
        assert np.array_equal(dev.values, vals)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_features_long_rows_warp_path(seed):
    """Rows longer than the per-thread limit (k_features hands them to a
    warp): runs of consecutive columns crossing 32-entry chunk boundaries,
    runs that start a row, single-entry gaps, very long dense rows and empty
    rows between them — aggregates equal the oracle's exactly."""
    rng = np.random.default_rng(seed)
    n = 3000
    rows = []
    for i in range(n):
        kind = rng.integers(0, 5)
        if kind == 0:
            rows.append(np.array([], dtype=np.int64))
        elif kind == 1:                          # short random row
            rows.append(np.unique(rng.integers(0, n, size=rng.integers(1, 20))))
        elif kind == 2:                          # long row of consecutive blocks
            starts = np.sort(rng.choice(n - 200, size=rng.integers(2, 6), replace=False))
            blk = [np.arange(s0, s0 + rng.integers(1, 150)) for s0 in starts]
            rows.append(np.unique(np.concatenate(blk)))
        elif kind == 3:                          # very long random row
            rows.append(np.unique(rng.integers(0, n, size=rng.integers(65, 1500))))
        else:                                    # one long consecutive run
            s0 = int(rng.integers(0, n - 700))
            rows.append(np.arange(s0, s0 + int(rng.integers(60, 700))))
    ptr = np.zeros(n + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([r.size for r in rows])
    cols = np.concatenate(rows).astype(np.int64)
    vals = np.ones(cols.size)
    A = P.CsrMatrix(n, n, ptr, cols, vals)
    got = P.extract_features(A)
    assert got.to_array().tolist() == O.features(O.OCsr(n, n, ptr, cols, vals))


@pytest.mark.parametrize("nd", [70, 300, 1200])
def test_dia_conversion_long_rows_warp_path(nd):
    """Banded rows longer than 64 entries (the diagonal bitmap marks them by
    a warp): the DIA offsets and data equal the oracle conversion exactly."""
    rng = np.random.default_rng(nd)
    n = 4000
    offs = np.unique(np.concatenate([[0], rng.integers(-1500, 1501, size=nd)]))
    nn, _, ptr, cols, vals = G.banded(n, offs.tolist(), seed=nd, diagonal_boost=2.0 * len(offs))
    A = P.CsrMatrix(nn, nn, ptr, cols, vals)
    D = P.convert(A, P.FormatTag.DIA)
    ref = O.convert(O.OCsr(nn, nn, ptr, cols, vals), "DIA")
    assert np.array_equal(np.asarray(D.offsets), np.asarray(ref.offsets))
    assert np.array_equal(np.asarray(D.data), np.asarray(ref.data))
