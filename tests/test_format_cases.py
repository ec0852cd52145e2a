"""The reference's container tests (tests/test_formats.py:16-50, 120-140):
host-side construction validation with the same error classes/messages,
from_triplets sorting and duplicate summation, frozen arrays; the
conversion and SpMV cases run on the GPU through the device containers."""
import numpy as np
import pytest

from paper_2411_10143_b200 import CooMatrix, CsrMatrix, FormatTag, convert


def entry_set(m):
    return {(int(r), int(c), float(v)) for r, c, v in zip(m.rows, m.cols, m.values)}


def identity_coo(n=3):
    return CooMatrix(n, n, np.arange(n), np.arange(n), np.ones(n))


class TestConstruction:
    def test_coo_rejects_unsorted(self):
        with pytest.raises(ValueError, match="sorted"):
            CooMatrix(2, 2, [1, 0], [0, 0], [1.0, 1.0])

    def test_coo_rejects_duplicates(self):
        with pytest.raises(ValueError):
            CooMatrix(2, 2, [0, 0], [1, 1], [1.0, 2.0])

    def test_coo_rejects_out_of_range(self):
        with pytest.raises(ValueError, match="out of range"):
            CooMatrix(2, 2, [0], [5], [1.0])

    def test_coo_rejects_nonfinite(self):
        with pytest.raises(ValueError, match="finite"):
            CooMatrix(2, 2, [0], [0], [np.inf])

    def test_from_triplets_sorts_and_sums(self):
        m = CooMatrix.from_triplets(2, 2, [1, 0, 1], [0, 1, 0], [1.0, 2.0, 3.0], sum_duplicates=True)
        assert entry_set(m) == {(0, 1, 2.0), (1, 0, 4.0)}

    def test_csr_rejects_bad_row_ptr(self):
        with pytest.raises(ValueError):
            CsrMatrix(2, 2, [0, 2], [0, 1], [1.0, 1.0])

    def test_csr_rejects_decreasing_columns(self):
        with pytest.raises(ValueError, match="strictly increasing"):
            CsrMatrix(1, 3, [0, 2], [2, 0], [1.0, 1.0])

    def test_arrays_are_immutable(self):
        m = identity_coo()
        with pytest.raises(ValueError):
            m.values[0] = 5.0


@pytest.mark.gpu
class TestDeviceConvert:
    def test_identity_to_csr(self):
        csr = convert(identity_coo(), FormatTag.CSR)
        assert np.asarray(csr.row_ptr).tolist() == [0, 1, 2, 3]
        assert np.asarray(csr.col_idx).tolist() == [0, 1, 2]

    def test_all_ones_to_ell_has_no_padding(self):
        r, c = np.nonzero(np.ones((2, 3)))
        ell = convert(CooMatrix(2, 3, r, c, np.ones(6)), FormatTag.ELL)
        assert ell.width == 3
        assert (np.asarray(ell.col_idx) < 3).all()

    def test_identity_to_dia_single_offset(self):
        dia = convert(identity_coo(4), FormatTag.DIA)
        assert np.asarray(dia.offsets).tolist() == [0]

    def test_from_triplets_device_matches_host(self):
        rng = np.random.default_rng(5)
        r = rng.integers(0, 50, 2000)
        c = rng.integers(0, 60, 2000)
        v = rng.standard_normal(2000)
        host = CooMatrix.from_triplets(50, 60, r, c, v, sum_duplicates=True)
        import ctypes

        from paper_2411_10143_b200 import _lib
        from paper_2411_10143_b200.formats import _new_handle
        r64, c64 = np.ascontiguousarray(r, np.int64), np.ascontiguousarray(c, np.int64)
        dev = CooMatrix._wrap(_new_handle(_lib.lib().svb_coo_from_triplets, 50, 60, 2000, r64.ctypes.data,
                                          c64.ctypes.data, v.ctypes.data, 1, None))
        for a, b in ((dev.rows, host.rows), (dev.cols, host.cols), (dev.values, host.values)):
            assert np.array_equal(np.asarray(a), np.asarray(b))
        del ctypes
