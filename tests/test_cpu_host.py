"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, and the host-side logic (config space, cascade via the compiled
forest, mailbox, feature formulas, LibC chunk bounds) matches the reference
contract.  No CUDA call is made here."""
import re
import threading
import time
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from golden_io import cascade_doc, case, case_names

import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import _lib
from paper_2411_10143_b200.features import features_from_aggregates
from paper_2411_10143_b200.formats import hyb_split_width
from paper_2411_10143_b200.solver import ConfigMailbox, _Update

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "spmvtune_b200.h").read_text()
    return sorted(set(re.findall(r"\b(svb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing
    assert sorted(_lib.exported_symbols()) == declared
    assert lib.svb_abi_version() == 1


def test_config_space_matches_reference_order():
    toks = [c.token() for c in P.enumerate_configs()]
    assert toks == list(O.TOKENS)
    assert P.enumerate_configs()[0] == P.DEFAULT_CONFIG
    for t in toks:
        assert P.SpmvConfig.from_token(t).token() == t
    with pytest.raises(P.UnsupportedConfigError):
        P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_A)
    with pytest.raises(P.UnsupportedConfigError):
        P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_A, 3)
    with pytest.raises(P.UnsupportedConfigError):
        P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_B)
    with pytest.raises(P.UnsupportedConfigError):
        P.SpmvConfig(P.FormatTag.COO, P.Library.LIB_A, 2)


def test_compiled_cascade_matches_reference_models():
    """The C++ forest evaluator reproduces the reference's labels AND
    float64 scores on >= 5000 rows of the shipped models."""
    doc = cascade_doc()
    models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
    by_name = {"FORMAT": models.format_model, "COO-LIB": models.coo_lib_model,
               "CSR-LIB": models.csr_lib_model, "ELL-LIB": models.ell_lib_model,
               "CSR-TPV": models.csr_tpv_model}
    total = 0
    for name, data in doc["models"].items():
        for row, lab, sc in zip(data["rows"], data["labels"], data["scores"]):
            got, scores = by_name[name].predict(np.asarray(row))
            assert got == lab
            assert scores.tolist() == sc
            total += 1
    assert total >= 5000
    for entry in doc["cascade"]:
        decisions = []
        final = P.cascade_predict(models, np.asarray(entry["row"]), decisions.append)
        assert final.token() == entry["final"]
        assert [d.implied_config().token() for d in decisions] == entry["decisions"]
        assert [d.stage.value for d in decisions] == entry["stages"]


def test_cascade_median_latency_under_budget():
    """Reference gate: full cascade median <= 1 ms (test_inference.py:271-291)."""
    models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
    x = np.asarray(cascade_doc()["cascade"][0]["row"])
    P.cascade_predict(models, x)
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        P.cascade_predict(models, x)
        ts.append(time.perf_counter() - t0)
    assert np.median(ts) <= 1e-3


@pytest.mark.parametrize("name", case_names())
def test_feature_formulas_bit_exact(name):
    c = case(name)
    csr = O.coo_to_csr(O.OCoo(int(c["nrows"]), int(c["ncols"]), c["coo_rows"], c["coo_cols"],
                              c["coo_vals"]))
    a = O.feature_aggregates(csr)
    agg = (a["sum_r"], a["sum_r2"], a["max_r"], a["min_r"], a["span"], a["runs"], a["ndiag"])
    fv = features_from_aggregates(csr.nrows, csr.ncols, int(csr.cols.size), agg)
    assert fv.to_array().tolist() == c["features"].tolist()


def test_hyb_split_width_goldens():
    # formats test goldens (reference test_formats.py:111-116)
    assert hyb_split_width(np.array([1, 1, 9])) == 1
    assert hyb_split_width(np.array([3, 5, 9])) == 5
    assert hyb_split_width(np.array([2, 2, 2, 2])) == 2
    assert hyb_split_width(np.array([0, 0, 7])) == 0
    rng = np.random.default_rng(1)
    for _ in range(200):
        lens = rng.integers(0, 50, size=int(rng.integers(1, 40)))
        assert hyb_split_width(lens) == O.hyb_width(lens)


def test_merge_bounds_formula_matches_numpy_linspace():
    """csrc/spmv.cu:merge_bounds restates np.linspace(..., dtype=int64):
    floor(c * (nnz/chunks)) with the last edge pinned to nnz."""
    import math
    rng = np.random.default_rng(3)
    cases = [(n, w) for n in (1, 2, 3, 7, 100, 1001, 65537, 35976004, 5812581592)
             for w in (1, 3, 4, 7, 64, 148, 1000)]
    cases += [(int(rng.integers(1, 10**9)), int(rng.integers(1, 5000))) for _ in range(300)]
    for nnz, workers in cases:
        chunks = min(workers, nnz)
        step = nnz / chunks
        mine = [math.floor(c * step) for c in range(chunks)] + [nnz]
        assert mine == O.merge_bounds(nnz, workers).tolist(), (nnz, workers)


class TestMailbox:
    cfg_a = P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_B)
    cfg_b = P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_C)

    def test_last_writer_wins(self):
        box = ConfigMailbox()
        box.publish(_Update(self.cfg_a, None, 0.0))
        box.publish(_Update(self.cfg_b, None, 0.0))
        assert box.poll(1).config == self.cfg_b
        assert box.poll(1) is None

    def test_gated_visibility(self):
        box = ConfigMailbox(expected_gates=[3])
        box.publish(_Update(self.cfg_a, None, 0.0))
        assert box.poll(2) is None
        assert box.poll(3).config == self.cfg_a

    def test_gated_poll_waits_for_late_publish(self):
        box = ConfigMailbox(expected_gates=[0])

        def later():
            time.sleep(0.05)
            box.publish(_Update(self.cfg_a, None, 0.0))

        t = threading.Thread(target=later)
        t.start()
        assert box.poll(1, timeout=5.0).config == self.cfg_a
        t.join()

    def test_tombstone_releases_gate(self):
        box = ConfigMailbox(expected_gates=[0])
        box.publish(_Update(None, None, 0.0))
        assert box.poll(5) is None


def test_params_validation():
    with pytest.raises(ValueError):
        P.GmresParams(restart_m=0)
    with pytest.raises(ValueError):
        P.GmresParams(tol=0.0)
    with pytest.raises(ValueError):
        P.GmresParams(tol=2.0)
    with pytest.raises(ValueError):
        P.GmresParams(rhs="zeros")


def test_host_validation_messages():
    with pytest.raises(ValueError, match="sorted"):
        P.CooMatrix(2, 2, [1, 0], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="out of range"):
        P.CooMatrix(2, 2, [0], [5], [1.0])
    with pytest.raises(ValueError, match="finite"):
        P.CooMatrix(2, 2, [0], [0], [np.inf])
    with pytest.raises(ValueError, match="strictly increasing"):
        P.CsrMatrix(1, 3, [0, 2], [2, 0], [1.0, 1.0])
    m = P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3))
    with pytest.raises(ValueError):
        m.values[0] = 5.0
    t = P.CooMatrix.from_triplets(2, 2, [1, 0, 1], [0, 1, 0], [1.0, 2.0, 3.0], sum_duplicates=True)
    assert set(zip(t.rows.tolist(), t.cols.tolist(), t.values.tolist())) == {(0, 1, 2.0), (1, 0, 4.0)}


def test_no_oracle_import_in_product():
    """The product package must never reach the CPU oracle."""
    for p in (ROOT / "paper_2411_10143_b200").rglob("*.py"):
        text = p.read_text()
        assert "import oracle" not in text and "from oracle" not in text, p


def test_native_mailbox_and_driver_argument_checks_on_host():
    """The C-ABI mailbox needs no GPU; the native drivers reject bad
    arguments before touching the device."""
    import ctypes
    from paper_2411_10143_b200 import _lib
    mb = P.NativeMailbox()
    assert mb.finished is False
    L = _lib.load()
    rep = _lib.SolveReportC()
    sp = _lib.SolveParams(30, 10, 1e-8)
    st = L.svb_gmres_run(None, _lib.SvbConfig(1, 1, 0, 1), None, None, ctypes.byref(sp), None, None,
                         None, None, 0, ctypes.byref(rep))
    assert st == _lib.INVALID and "null argument" in _lib.last_error()
    sp0 = _lib.SolveParams(0, 10, 1e-8)
    st = L.svb_gmres_run(None, _lib.SvbConfig(1, 1, 0, 1), None, None, ctypes.byref(sp0), None, None,
                         None, None, 0, ctypes.byref(rep))
    assert st == _lib.INVALID and "restart_m" in _lib.last_error()
    with pytest.raises(ValueError):
        P.native_solve("bicgstab", None)
    del mb


def test_native_loop_eligibility():
    """Stock executors run the C++ solver loop; probes, plugin executors and
    device-kept solutions keep the Python loop (solver._native_eligible)."""
    from paper_2411_10143_b200 import solver as S
    ex = S.SpmvExecutor.__new__(S.SpmvExecutor)
    p = S.GmresParams()
    assert S._native_eligible(ex, None, p, None) == (S._LOOP == "native")
    assert not S._native_eligible(ex, None, p, lambda it, c: None)

    class Plugin(S.SpmvExecutor):
        def matvec(self, x):
            return x

    assert not S._native_eligible(Plugin.__new__(Plugin), None, p, None)
    with S.DeviceOptions(keep_solution_on_device=True):
        assert not S._native_eligible(ex, None, p, None)


def test_bench_stdout_carries_only_the_json_line():
    """bench.py's measuring process keeps fd 1 for its JSON line; native
    writes to stdout (NCCL's version banner) and Python prints go to stderr."""
    import subprocess
    import sys
    from pathlib import Path
    code = ("import os, sys\nsys.argv = ['bench.py']\nimport bench\nbench._claim_stdout()\n"
            "print('python noise')\nos.write(1, b'native noise\\n')\nbench.emit({'metric': 'x', 'value': 1})\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       cwd=Path(__file__).resolve().parent.parent, timeout=120)
    assert p.returncode == 0, p.stderr[-1000:]
    assert p.stdout == '{"metric": "x", "value": 1}\n'
    assert "native noise" in p.stderr and "python noise" in p.stderr
