"""The reference's labelling / dataset tests (tests/test_bench.py:112-266)
against this package: argmin labels per stage with exact ties to the lower
config index, routing of a matrix's feature row into the stage datasets, and
(on the GPU) build_dataset's CSV layout, routing counts, skip-and-log of bad
files and the resumable timing cache."""
import json

import numpy as np
import pytest

from paper_2411_10143_b200 import (FEATURE_NAMES, SpmvTuneError, TimingRecord, enumerate_configs,
                                   label_from_times, route_labels)

ALL = [c.token() for c in enumerate_configs()]
LANES = [f"CSR/LibA/{w}" for w in (2, 4, 8, 16, 32)]


def synthetic_times(rng, tie_fraction=0.0, dia_inapplicable=False):
    times = {t: float(rng.uniform(1e-6, 1e-3)) for t in ALL}
    if tie_fraction and rng.random() < tie_fraction:
        a, b = rng.choice(len(ALL), size=2, replace=False)
        times[ALL[b]] = times[ALL[a]]
    if dia_inapplicable:
        times["DIA/LibA"] = None
    return times


def brute_force(times):
    def argmin(pairs):
        best = None
        for label, t in pairs:
            if t is not None and (best is None or t < best[1]):
                best = (label, t)
        return best[0] if best else None
    lanes = [times[t] for t in LANES if times[t] is not None]
    csr_a = min(lanes) if lanes else None
    return {"format": argmin([("COO", times["COO/LibA"]), ("CSR", csr_a), ("ELL", times["ELL/LibA"]),
                              ("DIA", times["DIA/LibA"]), ("HYB", times["HYB/LibA"])]),
            "coo_lib": argmin([("LibA", times["COO/LibA"]), ("LibB", times["COO/LibB"])]),
            "csr_lib": argmin([("LibA", csr_a), ("LibB", times["CSR/LibB"]), ("LibC", times["CSR/LibC"])]),
            "ell_lib": argmin([("LibA", times["ELL/LibA"]), ("LibC", times["ELL/LibC"])]),
            "tpv": argmin([(t.rsplit("/", 1)[1], times[t]) for t in LANES])}


def test_argmin_oracle_random_tables():
    rng = np.random.default_rng(33)
    for i in range(100):
        times = synthetic_times(rng, tie_fraction=0.5, dia_inapplicable=(i % 7 == 0))
        got, want = label_from_times(times), brute_force(times)
        assert (got.format, got.coo_lib, got.csr_lib, got.ell_lib, got.tpv) == \
            (want["format"], want["coo_lib"], want["csr_lib"], want["ell_lib"], want["tpv"])


def test_exact_tie_takes_lower_config_index():
    lab = label_from_times({t: 1.0 for t in ALL})
    assert (lab.format, lab.coo_lib, lab.csr_lib, lab.ell_lib, lab.tpv) == ("COO", "LibA", "LibA", "LibA", "2")


def test_dia_fastest_routes_nowhere():
    times = synthetic_times(np.random.default_rng(4))
    times["DIA/LibA"] = 1e-9
    lab = label_from_times(times)
    assert lab.format == "DIA" and route_labels(lab) == {"FORMAT": "DIA"}


def test_csr_liba_routes_to_lane_dataset():
    times = {t: 1.0 for t in ALL}
    times["CSR/LibA/8"] = 0.1
    lab = label_from_times(times)
    routed = route_labels(lab)
    assert lab.format == "CSR" and lab.csr_lib == "LibA" and lab.tpv == "8"
    assert set(routed) == {"FORMAT", "CSR-LIB", "CSR-TPV"} and routed["CSR-TPV"] == "8"


def test_csr_other_lib_skips_lane_dataset():
    times = {t: 1.0 for t in ALL}
    times["CSR/LibC"] = 0.05
    for t in LANES:
        times[t] = 0.08
    lab = label_from_times(times)
    assert lab.format == "CSR" and lab.csr_lib == "LibC"
    assert set(route_labels(lab)) == {"FORMAT", "CSR-LIB"}


def test_empty_directory_raises(tmp_path):
    from paper_2411_10143_b200 import build_dataset
    (tmp_path / "none").mkdir()
    with pytest.raises(SpmvTuneError, match="no .mtx"):
        build_dataset(tmp_path / "none", tmp_path / "out")


# ---------------------------------------------------------------------------
# build_dataset end to end (features on the device)
# ---------------------------------------------------------------------------
def _write_mtx(path, n, rows, cols, vals):
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{n} {n} {len(rows)}\n")
        for r, c, v in zip(rows, cols, vals):
            fh.write(f"{r + 1} {c + 1} {float(v)!r}\n")


@pytest.fixture
def matrix_dir(tmp_path):
    d = tmp_path / "matrices"
    d.mkdir()
    rng = np.random.default_rng(1)
    for i in range(6):
        n = int(rng.integers(10, 41))
        dense = (rng.random((n, n)) < 0.3) * rng.uniform(-1, 1, (n, n))
        dense[np.arange(n), np.arange(n)] += n
        r, c = np.nonzero(dense)
        _write_mtx(d / f"m{i}.mtx", n, r, c, dense[r, c])
    return d


def fixed_timer(fastest):
    def timer(matrix, matrix_id):
        times = {t: 1.0 for t in ALL}
        times.update(fastest.get(matrix_id, {}))
        return TimingRecord(matrix_id=matrix_id, times=times, runs=1, warmups=0, workers=1)
    return timer


@pytest.mark.gpu
def test_routing_row_counts(matrix_dir, tmp_path):
    from paper_2411_10143_b200 import build_dataset
    out = tmp_path / "out"
    fastest = {"m0": {"DIA/LibA": 0.1}, "m1": {"COO/LibB": 0.1}, "m2": {"CSR/LibA/16": 0.1},
               "m3": {"CSR/LibA/2": 0.2, "CSR/LibC": 0.1}, "m4": {"ELL/LibA": 0.2, "ELL/LibC": 0.1},
               "m5": {"HYB/LibA": 0.1}}
    counts = build_dataset(matrix_dir, out, timer=fixed_timer(fastest))
    assert counts == {"FORMAT": 6, "COO-LIB": 1, "CSR-LIB": 2, "ELL-LIB": 1, "CSR-TPV": 1}
    lines = [ln for ln in (out / "FORMAT.csv").read_text().splitlines() if ln and not ln.startswith("#")]
    assert lines[0] == ",".join(FEATURE_NAMES) + ",label" and len(lines) == 7
    assert sorted(ln.rsplit(",", 1)[1] for ln in lines[1:]) == ["COO", "CSR", "CSR", "DIA", "ELL", "HYB"]
    tpv = [ln for ln in (out / "CSR-TPV.csv").read_text().splitlines() if ln and not ln.startswith("#")]
    assert tpv[1].endswith(",16")


@pytest.mark.gpu
def test_bad_matrix_skipped_and_logged(matrix_dir, tmp_path, caplog):
    from paper_2411_10143_b200 import build_dataset
    (matrix_dir / "broken.mtx").write_text("%%MatrixMarket junk\n")
    with caplog.at_level("WARNING"):
        counts = build_dataset(matrix_dir, tmp_path / "out", timer=fixed_timer({}))
    assert counts["FORMAT"] == 6
    assert any("broken" in rec.message for rec in caplog.records)


@pytest.mark.gpu
def test_resumable_cache(matrix_dir, tmp_path):
    from paper_2411_10143_b200 import build_dataset
    calls = []

    def timer(matrix, matrix_id):
        calls.append(matrix_id)
        return TimingRecord(matrix_id=matrix_id, times={t: 1.0 for t in ALL}, runs=200, warmups=10,
                            workers=4)
    build_dataset(matrix_dir, tmp_path / "out", runs=200, warmups=10, workers=4, timer=timer)
    assert len(calls) == 6
    build_dataset(matrix_dir, tmp_path / "out", runs=200, warmups=10, workers=4, timer=timer)
    assert len(calls) == 6
    assert json.loads((tmp_path / "out" / "cache" / "m0.json").read_text())["matrix_id"] == "m0"
