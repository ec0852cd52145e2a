"""Matrix Market ingest (reference tests/test_mmio.py cases): the host
parser on CPU; the native multi-threaded parser + device from_triplets on the
GPU, on the same cases written to files and on a large generated file
(bit-exact against the host path, duplicates summed in reduceat order)."""
import numpy as np
import pytest

import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import MatrixMarketError, parse_matrix_market

IDENTITY = """%%MatrixMarket matrix coordinate real general
% 3x3 identity
3 3 3
1 1 1.0
2 2 1.0
3 3 1.0
"""

GOOD = {
    "identity": (IDENTITY, {(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)}),
    "symmetric": ("%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2.0\n2 1 5.0\n2 2 3.0\n",
                  {(0, 0, 2.0), (1, 0, 5.0), (0, 1, 5.0), (1, 1, 3.0)}),
    "pattern_dups": ("%%MatrixMarket matrix coordinate pattern general\n2 2 3\n1 1\n2 2\n1 1\n",
                     {(0, 0, 2.0), (1, 1, 1.0)}),
    "integer": ("%%MatrixMarket matrix coordinate integer general\n1 2 2\n1 1 7\n1 2 -3\n",
                {(0, 0, 7.0), (0, 1, -3.0)}),
    "sym_diag": ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 4.0\n", {(0, 0, 4.0)}),
}

BAD = {
    "complex": ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n", "complex"),
    "banner": ("%%NotMatrixMarket whatever\n1 1 0\n", "banner"),
    "symmetry": ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1.0\n", "symmetry"),
    "array": ("%%MatrixMarket matrix array real general\n1 1\n1.0\n", "coordinate"),
    "range": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of range"),
    "truncated": ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "truncated"),
    "extra": ("%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n1 1 2.0\n", "more entries"),
    "fields": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "expected 3 fields"),
    "malformed": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", "malformed fields"),
    "size": ("%%MatrixMarket matrix coordinate real general\n2 2\n1 1 1.0\n", "size line"),
}


def entry_set(m):
    return {(int(r), int(c), float(v)) for r, c, v in zip(m.rows, m.cols, m.values)}


@pytest.mark.parametrize("name", sorted(GOOD))
def test_host_parser_cases(name):
    text, want = GOOD[name]
    assert entry_set(parse_matrix_market(text)) == want


@pytest.mark.parametrize("name", sorted(BAD))
def test_host_parser_errors(name):
    text, match = BAD[name]
    with pytest.raises(MatrixMarketError, match=match):
        parse_matrix_market(text)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOOD))
def test_native_loader_cases(tmp_path, name):
    text, want = GOOD[name]
    f = tmp_path / f"{name}.mtx"
    f.write_text(text)
    m = P.load_matrix_market(f)
    assert entry_set(m) == want
    h = parse_matrix_market(text)
    assert np.array_equal(np.asarray(m.rows), np.asarray(h.rows))
    assert np.array_equal(np.asarray(m.cols), np.asarray(h.cols))
    assert np.array_equal(np.asarray(m.values), np.asarray(h.values))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(BAD))
def test_native_loader_errors(tmp_path, name):
    text, match = BAD[name]
    f = tmp_path / f"{name}.mtx"
    f.write_text(text)
    with pytest.raises(MatrixMarketError, match=match):
        P.load_matrix_market(f)


@pytest.mark.gpu
@pytest.mark.parametrize("threads", [1, 7])
def test_native_loader_large_matches_host(tmp_path, threads):
    """600 K random entries (duplicates, comments, blank lines, symmetric):
    same sorted arrays as the host parser (reduceat-order duplicate sums),
    and the first bad entry reported when one is planted late in the file."""
    rng = np.random.default_rng(3)
    n, k = 5000, 600_000
    r = rng.integers(1, n + 1, size=k)
    c = rng.integers(1, n + 1, size=k)
    v = rng.standard_normal(k)
    lines = ["%%MatrixMarket matrix coordinate real symmetric", "% generated", f"{n} {n} {k}"]
    for i in range(k):
        lines.append(f"{r[i]} {c[i]} {float(v[i])!r}")
        if i % 50_000 == 0:
            lines.append("% comment")
            lines.append("")
    text = "\n".join(lines) + "\n"
    f = tmp_path / "big.mtx"
    f.write_text(text)
    m = P.load_matrix_market(f, threads=threads)
    h = parse_matrix_market(text)
    assert m.nnz == h.nnz
    for a, b in ((m.rows, h.rows), (m.cols, h.cols), (m.values, h.values)):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    bad = lines[:]
    bad[3 + 400_000] = "1 2"
    bad[3 + 500_000] = f"{n + 7} 1 1.0"
    f.write_text("\n".join(bad) + "\n")
    with pytest.raises(MatrixMarketError) as e1:
        P.load_matrix_market(f, threads=threads)
    with pytest.raises(MatrixMarketError) as e2:
        parse_matrix_market("\n".join(bad) + "\n")
    assert str(e1.value) == str(e2.value)
