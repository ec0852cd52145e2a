"""CLI on the B200 backend (reference cli.py): report formatting and exit
codes on CPU; dataset / suite / compare end to end on the GPU."""
import json

import numpy as np
import pytest

from paper_2411_10143_b200 import cli


def _fake_compare(matrix_id, d, s, a, final="DIA/LibA", swap=3):
    rep = lambda w, tl: {"converged": True, "iterations": 10, "residual_history": [],  # noqa: E731
                         "config_timeline": tl, "advisor_outcome": "completed",
                         "final_residual": 1e-9, "wall_seconds": w}
    tl0 = [{"iteration": 1, "config": "CSR/LibA/32", "swap_cost_seconds": 0.0}]
    return {"matrix_id": matrix_id, "default": rep(d, tl0), "sequential": rep(s, tl0),
            "async": rep(a, tl0 + [{"iteration": swap, "config": final, "swap_cost_seconds": 1e-3}]),
            "speedup_sequential": d / s, "speedup_async": d / a}


def test_report_table_csv_and_geomean(tmp_path, capsys):
    (tmp_path / "a_compare.json").write_text(json.dumps(_fake_compare("a", 2.0, 1.0, 0.5)))
    (tmp_path / "b_compare.json").write_text(json.dumps(_fake_compare("b", 1.0, 1.0, 1.0, "CSR/LibB", 2)))
    out = tmp_path / "sum.csv"
    assert cli.main(["report", str(tmp_path), "--out", str(out)]) == 0
    text = capsys.readouterr().out
    assert "a " in text and "DIA/LibA" in text and "geometric mean" in text
    assert "2.00" in text                       # geomean of async speedups 4 and 1
    rows = out.read_text().splitlines()
    assert rows[0].split(",") == ["matrix", "default_s", "sequential_s", "async_s", "speedup_sequential",
                                  "speedup_async", "final_config", "swap_iterations"]
    assert len(rows) == 3 and rows[1].endswith(",DIA/LibA,3")


def test_exit_codes(tmp_path):
    assert cli.main(["report", str(tmp_path)]) == cli.EXIT_DATA          # no compare files
    assert cli.main(["compare", str(tmp_path / "missing.mtx"), "--models", "x"]) == cli.EXIT_DATA
    with pytest.raises(SystemExit) as exc:
        cli.main(["solve"])                                              # usage error
    assert exc.value.code == 2


def test_suite_generator_families():
    ids = [mid for mid, _ in _shapes()]
    fams = sorted({i.rsplit("_", 1)[0] for i in ids})
    assert fams == ["banded", "convdiff9", "poisson2d", "powerlaw", "random"]
    assert len(ids) == 10


def _shapes():
    # host-only view of the suite (the generator builds CsrMatrix objects,
    # which stay host-side until first device use)
    return list(cli.suite_matrices(per_family=2, scale=0.0005))


def test_random_dd_is_diagonally_dominant():
    n, _, ptr, cols, vals = cli._random_dd(200, 6, 3)
    for i in range(n):
        s, e = ptr[i], ptr[i + 1]
        c, v = cols[s:e], vals[s:e]
        assert np.all(np.diff(c) > 0)
        d = v[c == i][0]
        assert d > np.abs(v[c != i]).sum()


@pytest.mark.gpu
def test_dataset_suite_and_report_on_gpu(tmp_path, capsys):
    import os
    import paper_2411_10143_b200 as P
    models = os.path.join(os.path.dirname(__file__), "golden", "models")
    mats = list(cli.suite_matrices(per_family=1, scale=0.002))
    counts = P.build_dataset(None, tmp_path / "ds", runs=3, warmups=1, matrices=mats)
    assert counts["FORMAT"] == len(mats)
    hdr = (tmp_path / "ds" / "FORMAT.csv").read_text().splitlines()
    assert hdr[0].startswith("# host=") and hdr[1].split(",")[-1] == "label"
    assert len(hdr) == 2 + len(mats)
    assert len(list((tmp_path / "ds" / "cache").glob("*.json"))) == len(mats)
    assert cli.main(["suite", "--models", models, "--out", str(tmp_path / "cmp"), "--per-family", "1",
                     "--scale", "0.002", "--max-iters", "300"]) == 0
    assert cli.main(["report", str(tmp_path / "cmp")]) == 0
    assert "geometric mean" in capsys.readouterr().out
