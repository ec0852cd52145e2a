"""GPU parity: the 13 SpMV kernels against the reference's own outputs.

Every deterministic configuration must be BIT-IDENTICAL to the golden y the
reference produced (tests/golden, generated from /root/reference); COO/LibB
(atomic scatter, nondeterministic in the reference too) is held to the
reference's 1e-8 bar.  Larger matrices are checked against the CPU oracle
bit-for-bit, fp32 against fp64 at fp32 tolerance.
"""
import os

import numpy as np
import pytest

import oracle as O
from golden_io import case, case_names, spmv_keys

import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import device, generators as G

pytestmark = pytest.mark.gpu
ATOMIC = P.SpmvConfig(P.FormatTag.COO, P.Library.LIB_B)


def coo_of(c):
    return P.CooMatrix(int(c["nrows"]), int(c["ncols"]), c["coo_rows"], c["coo_cols"], c["coo_vals"])


def rel(got, want):
    s = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (s if s else 1.0)


@pytest.mark.parametrize("name", case_names())
def test_golden_bit_exact(name):
    c = case(name)
    coo = coo_of(c)
    reps = {}
    for tok, w in spmv_keys(c):
        cfg = P.SpmvConfig.from_token(tok)
        if cfg.format not in reps:
            reps[cfg.format] = P.convert(coo, cfg.format)
        got = P.execute_spmv(cfg, reps[cfg.format], c["x"], workers=w)
        want = c[f"y|{tok}|{w}"]
        assert np.array_equal(got, want), (tok, w, np.max(np.abs(got - want)))
        # sign of zero included: the kernels mirror numpy's -0.0 handling too
        assert np.array_equal(np.signbit(got), np.signbit(want)), (tok, w)
    got = P.execute_spmv(ATOMIC, coo, c["x"])
    assert rel(got, c["y_reference"]) <= 1e-8
    csr = reps.get(P.FormatTag.CSR) or P.convert(coo, P.FormatTag.CSR)
    assert np.array_equal(P.spmv_reference(csr, c["x"]), c["y_reference"])


@pytest.mark.parametrize("gen", ["poisson", "convdiff", "powerlaw", "laplace27"])
def test_larger_matrices_against_oracle(gen):
    n, m, ptr, cols, vals = {
        "poisson": lambda: G.poisson2d(300),
        "convdiff": lambda: G.convdiff9(200),
        "powerlaw": lambda: G.powerlaw_spd(60000, seed=7),
        "laplace27": lambda: G.laplace27(30),
    }[gen]()
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    ocsr = O.OCsr(n, m, ptr, cols, vals)
    x = np.random.default_rng(11).uniform(-1.0, 1.0, size=m)
    reps = {"CSR": ocsr, "COO": O.csr_to_coo(ocsr)}
    for fmt in ("ELL", "DIA", "HYB"):
        try:
            reps[fmt] = O.convert(ocsr, fmt)
        except O.OracleInapplicable:
            pass
    for cfg in P.enumerate_configs():
        if cfg.format.value not in reps or cfg == ATOMIC:
            continue
        rep = P.convert(csr, cfg.format)
        for w in ((1, 4, 148) if cfg.library is P.Library.LIB_C else (4,)):
            got = P.execute_spmv(cfg, rep, x, workers=w)
            want = O.spmv(cfg.token(), reps[cfg.format.value], x, workers=w)
            assert np.array_equal(got, want), (cfg.token(), w)
    got = P.execute_spmv(ATOMIC, P.convert(csr, P.FormatTag.COO), x)
    assert rel(got, O.spmv_sequential(ocsr, x)) <= 1e-12


def _skewed_csr(n=40000, seed=5):
    """Short rows, medium rows (warp path) and rows longer than MED_ROW (whole
    CTA): the row kernel then claims its tiles from the dynamic counter."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 20, size=n)
    lens[rng.choice(n, 40, replace=False)] = rng.integers(129, 1024, size=40)
    lens[rng.choice(n, 6, replace=False)] = [1025, 1500, 2049, 3000, 4100, 9000]
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    cols = np.concatenate([np.sort(rng.choice(n, int(k), replace=False)) for k in lens]).astype(np.int64)
    vals = rng.uniform(-1.0, 1.0, size=cols.size)
    return n, n, ptr, cols, vals


def test_dynamic_tile_claims_bit_exact_and_reset_across_launches_and_streams():
    """Matrices with rows > MED_ROW run the row kernel with dynamic tile
    claims (csrc/spmv.cu k_rows_pipe<..., DYN>): every deterministic CSR/COO/
    HYB configuration stays bit-identical to the oracle, launch after launch
    and on two streams (the per-(handle, stream) counter resets itself)."""
    n, m, ptr, cols, vals = _skewed_csr()
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    ocsr = O.OCsr(n, m, ptr, cols, vals)
    reps = {"CSR": ocsr, "COO": O.csr_to_coo(ocsr), "HYB": O.convert(ocsr, "HYB")}
    x = np.random.default_rng(3).uniform(-1.0, 1.0, size=m)
    streams = [device.thread_stream(), device.Stream(0)]
    xds = [device.DeviceVector.from_numpy(x, s) for s in streams]
    for cfg in P.enumerate_configs():
        if cfg.format.value not in reps or cfg == ATOMIC:
            continue
        rep = P.convert(csr, cfg.format)
        want = O.spmv(cfg.token(), reps[cfg.format.value], x, workers=4)
        for k in range(6):
            s = streams[k % 2]
            got = P.execute_spmv(cfg, rep, xds[k % 2], workers=4, stream=s).to_numpy(s)
            assert np.array_equal(got, want), (cfg.token(), k)


FP32_TOL = 1e-5   # fp32 SpMV vs the fp64 result, relative 2-norm (fp32 values, x and sums)


@pytest.mark.parametrize("gen", ["powerlaw", "convdiff", "banded"])
def test_fp32_kernels_against_fp64(gen):
    """fp32 SpMV of every configuration the matrix admits (north star:
    "fp64/fp32 SpMV for every format") — DIA included on the banded and
    stencil matrices (the power-law one has too many diagonals)."""
    if gen == "powerlaw":
        n, m, ptr, cols, vals = G.powerlaw_spd(20000, seed=2)
    elif gen == "convdiff":
        n, m, ptr, cols, vals = G.convdiff9(150)
    else:
        n, m, ptr, cols, vals = G.banded(30000, [-700, -3, -1, 0, 2, 9, 1500], seed=4, diagonal_boost=3.0)
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    x = np.random.default_rng(5).uniform(0.5, 1.5, size=m)
    s = device.thread_stream()
    x32 = device.DeviceVector.from_numpy(x.astype(np.float32), s)
    x64 = device.DeviceVector.from_numpy(x, s)
    seen = set()
    for cfg in P.enumerate_configs():
        try:
            rep = P.convert(csr, cfg.format)
        except P.FormatInapplicableError:
            assert gen == "powerlaw" and cfg.format is P.FormatTag.DIA
            continue
        y64 = P.execute_spmv(cfg, rep, x64, stream=s).to_numpy(s)
        y32 = P.execute_spmv(cfg, rep, x32, stream=s).to_numpy(s)
        assert y32.dtype == np.float32
        assert rel(y32.astype(np.float64), y64) <= FP32_TOL, cfg.token()
        seen.add(cfg.format)
    assert len(seen) == (4 if gen == "powerlaw" else 5)


@pytest.mark.parametrize("n,offsets", [
    (20_000, [0]), (20_000, [-3, -1, 0, 1, 5]), (20_002, list(range(-13, 14))),
    (20_001, [-7, 0, 7]),                                   # odd rows: the thread-per-row kernel
    (65_536, list(range(-2000, 2001, 100))),                # 41 diagonals, wide reach: boundary tiles
    (33_000, list(range(-30, 31))),                         # 61 diagonals: above the staged-kernel limit
    (4_100, [-4099, -1, 0, 1, 4099])])                      # offsets touching the corners
def test_dia_staged_kernel_bit_exact(n, offsets):
    """The TMA-staged DIA kernel (k_dia_tma: tiles of every diagonal bulk
    copied through a shared-memory ring) against the oracle, fp64 bit-exact
    and fp32 within FP32_TOL, over interior, boundary and tail tiles."""
    nn, m, ptr, cols, vals = G.banded(n, offsets, seed=len(offsets), diagonal_boost=2.0)
    csr = P.CsrMatrix(nn, m, ptr, cols, vals)
    dia = P.convert(csr, P.FormatTag.DIA)
    cfg = P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)
    x = np.random.default_rng(n).uniform(-1.0, 1.0, size=m)
    want = O.spmv("DIA/LibA", O.convert(O.OCsr(nn, m, ptr, cols, vals), "DIA"), x)
    assert np.array_equal(P.execute_spmv(cfg, dia, x), want)
    s = device.thread_stream()
    y32 = P.execute_spmv(cfg, dia, device.DeviceVector.from_numpy(x.astype(np.float32), s), stream=s).to_numpy(s)
    assert rel(y32.astype(np.float64), want) <= FP32_TOL


def test_ell_strided_every_stride_bit_exact():
    """ELL/LibC with S = min(workers, width) from 1 to past the width: the
    compile-time-S kernels (S <= 16), the S >= width column sweep and the
    generic loop (S > 16) all reproduce the reference's strided partials."""
    n, m, ptr, cols, vals = G.banded(12_000, list(range(-11, 12)), seed=3, diagonal_boost=4.0)   # width 23
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    ell = P.convert(csr, P.FormatTag.ELL)
    oell = O.convert(O.OCsr(n, m, ptr, cols, vals), "ELL")
    cfg = P.SpmvConfig(P.FormatTag.ELL, P.Library.LIB_C)
    x = np.random.default_rng(9).uniform(-1.0, 1.0, size=m)
    assert ell.width == 23
    for w in list(range(1, 19)) + [22, 23, 24, 64]:
        assert np.array_equal(P.execute_spmv(cfg, ell, x, workers=w), O.spmv("ELL/LibC", oell, x, workers=w)), w


@pytest.mark.parametrize("n,offsets", [
    (40_000, [-201, -200, -199, -1, 0, 1, 199, 200, 201]),   # every offset residue mod 4
    (40_004, [-3, -2, -1, 0, 1, 2, 3]),
    (4_096, [-4095, -5, 0, 6, 4095]),                         # corners: the scalar edge path
    (40_001, [-7, 0, 7])])                                    # nrows % 4 != 0: the scalar kernel
def test_fp32_dia_bit_exact_against_float32_sweep(n, offsets):
    """fp32 DIA (k_dia_f32x4: 16-byte requests, four rows per thread) against
    the reference's diagonal sweep evaluated in float32 (each product and sum
    rounded to fp32, ascending offsets, out-of-range cells skipped)."""
    nn, m, ptr, cols, vals = G.banded(n, offsets, seed=n, diagonal_boost=2.0)
    dia = P.convert(P.CsrMatrix(nn, m, ptr, cols, vals), P.FormatTag.DIA)
    x32 = np.random.default_rng(n).uniform(-1.0, 1.0, size=m).astype(np.float32)
    data32 = np.asarray(dia.data).astype(np.float32)
    want = np.zeros(nn, dtype=np.float32)
    for k, off in enumerate(np.asarray(dia.offsets).tolist()):
        i0, i1 = max(0, -off), min(nn, m - off)
        if i0 < i1:
            want[i0:i1] = want[i0:i1] + data32[k, i0:i1] * x32[i0 + off:i1 + off]
    s = device.thread_stream()
    y32 = P.execute_spmv(P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A), dia,
                         device.DeviceVector.from_numpy(x32, s), stream=s).to_numpy(s)
    assert y32.dtype == np.float32 and np.array_equal(y32, want)


def test_ptr64_mode_is_what_the_environment_asks():
    """tests/test_gpu_scale.py re-runs this module with SPMVTUNE_FORCE_PTR64=1:
    the int64 row-pointer kernels must then really be the ones running."""
    n, m, ptr, cols, vals = G.poisson2d(20)
    A = P.CsrMatrix(n, m, ptr, cols, vals)
    forced = os.environ.get("SPMVTUNE_FORCE_PTR64") == "1"
    assert bool(A._device().info.ptr64) == forced
    assert bool(P.convert(P.to_coo(A), P.FormatTag.CSR)._device().info.ptr64) == forced


class TestDeviceOutValidation:
    """Raw-pointer kernels must never see a short, mistyped or strided
    buffer (silent device-memory corruption)."""

    def setup_method(self):
        n, m, ptr, cols, vals = G.poisson2d(12)
        self.A = P.CsrMatrix(n, m, ptr, cols, vals)
        self.cfg = P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_B)

    def test_short_or_mistyped_out(self):
        torch = pytest.importorskip("torch")
        x = torch.rand(self.A.ncols, dtype=torch.float64, device="cuda")
        for bad in (torch.empty(self.A.nrows - 1, dtype=torch.float64, device="cuda"),
                    torch.empty(self.A.nrows, dtype=torch.float32, device="cuda"),
                    torch.empty(self.A.nrows, dtype=torch.float16, device="cuda"),
                    np.empty(self.A.nrows)):
            with pytest.raises(ValueError):
                P.execute_spmv(self.cfg, self.A, x, out=bad)
        y = torch.full((self.A.nrows,), 7.0, dtype=torch.float64, device="cuda")
        assert P.execute_spmv(self.cfg, self.A, x, out=y) is y

    def test_bad_x(self):
        torch = pytest.importorskip("torch")
        with pytest.raises(ValueError):
            P.execute_spmv(self.cfg, self.A, torch.ones(self.A.ncols, dtype=torch.int64, device="cuda"))
        with pytest.raises(ValueError):
            P.execute_spmv(self.cfg, self.A, torch.rand(2 * self.A.ncols, dtype=torch.float64,
                                                        device="cuda")[::2])
        dv = device.DeviceVector(self.A.ncols, np.float64)
        with pytest.raises(ValueError):
            P.execute_spmv(self.cfg, self.A, dv, out=device.DeviceVector(self.A.nrows + 3))


def test_device_buffer_path_matches_host_path():
    n, m, ptr, cols, vals = G.convdiff9(64)
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    x = np.random.default_rng(1).uniform(0.5, 1.5, size=m)
    s = device.thread_stream()
    xd = device.DeviceVector.from_numpy(x, s)
    for cfg in P.enumerate_configs():
        if cfg == ATOMIC:
            continue
        rep = P.convert(csr, cfg.format)
        host = P.execute_spmv(cfg, rep, x)
        dev = P.execute_spmv(cfg, rep, xd, stream=s).to_numpy(s)
        assert np.array_equal(host, dev), cfg.token()


def test_torch_tensor_interop():
    torch = pytest.importorskip("torch")
    n, m, ptr, cols, vals = G.poisson2d(50)
    csr = P.CsrMatrix(n, m, ptr, cols, vals)
    x = torch.rand(m, dtype=torch.float64, device="cuda")
    cfg = P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_A, 8)
    y = P.execute_spmv(cfg, csr, x)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), P.execute_spmv(cfg, csr, x.cpu().numpy()))


class TestContract:
    def test_out_buffer_identity_and_refill(self):
        csr = P.convert(P.CooMatrix(4, 4, np.arange(4), np.arange(4), np.ones(4)), P.FormatTag.CSR)
        out = np.full(4, 7.0)
        got = P.execute_spmv(P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_B), csr, np.ones(4),
                             workers=2, out=out)
        assert got is out and out.tolist() == [1.0] * 4

    def test_format_mismatch(self):
        coo = P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3))
        with pytest.raises(P.UnsupportedConfigError, match="expects"):
            P.execute_spmv(P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_B), coo, np.ones(3))

    def test_dimension_mismatch(self):
        coo = P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3))
        with pytest.raises(ValueError, match="length"):
            P.execute_spmv(P.DEFAULT_CONFIG, coo, np.ones(4))

    def test_empty_matrix_all_configs(self):
        coo = P.CooMatrix(4, 5, [], [], [])
        for cfg in P.enumerate_configs():
            y = P.execute_spmv(cfg, P.convert(coo, cfg.format), np.ones(5))
            assert y.tolist() == [0.0] * 4, cfg.token()

    def test_lane32_identity(self):
        csr = P.convert(P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3)), P.FormatTag.CSR)
        got = P.execute_spmv(P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_A, 32), csr,
                             np.array([1.0, 2.0, 3.0]))
        assert got.tolist() == [1.0, 2.0, 3.0]

    def test_determinism(self):
        n, m, ptr, cols, vals = G.powerlaw_spd(30000, seed=9)
        csr = P.CsrMatrix(n, m, ptr, cols, vals)
        x = np.random.default_rng(2).uniform(0.5, 1.5, size=m)
        for cfg in P.enumerate_configs():
            if cfg == ATOMIC or cfg.format is P.FormatTag.DIA:
                continue
            rep = P.convert(csr, cfg.format)
            a = P.execute_spmv(cfg, rep, x)
            b = P.execute_spmv(cfg, rep, x)
            assert np.array_equal(a, b), cfg.token()
