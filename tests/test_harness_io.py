"""CPU tests of the input path and the report plumbing:
the native Matrix Market reader (ds_mm_read) against the reference reader's own
results on committed fixtures (tests/golden/make_golden_mtx.py), the report
emitters / parser (test_harness.py:177-200 patterns) and the CLI's usage errors."""
import math
import os

import numpy as np
import pytest

from paper_1511_07207_b200 import cli
from paper_1511_07207_b200.harness import (BenchRecord, MatrixMarketError, emit_report, parse_report_csv,
                                           read_matrix_market)

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden_mtx.npz"))
NAMES = [str(n) for n in G["names"]]


@pytest.mark.parametrize("name", NAMES)
def test_matrix_market_matches_reference(name):
    path = os.path.join(HERE, "golden", "mtx", name + ".mtx")
    if f"{name}_A" in G.files:
        A = read_matrix_market(path)
        ref = G[f"{name}_A"]
        assert A.shape == ref.shape and A.dtype == np.float64 and A.flags.f_contiguous
        np.testing.assert_array_equal(A, ref)
    else:
        with pytest.raises(MatrixMarketError) as e:
            read_matrix_market(path)
        assert e.value.line == int(G[f"{name}_err_line"])
        assert str(e.value) == str(G[f"{name}_err_msg"])  # the reference's exact message


def test_matrix_market_missing_file(tmp_path):
    with pytest.raises(FileNotFoundError):
        read_matrix_market(tmp_path / "nope.mtx")


def test_matrix_market_large_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    A = rng.uniform(-1, 1, (300, 200))
    p = tmp_path / "big.mtx"
    with open(p, "w") as fh:
        fh.write("%%MatrixMarket matrix array real general\n300 200\n")
        fh.write("".join(f"{float(v)!r}\n" for v in A.ravel(order="F")))
    np.testing.assert_array_equal(read_matrix_market(p), A)


def _recs():
    return [BenchRecord("cg", 256, "f64", "b200", 0.01, 12, True, 8.5e-9, 1.0),
            BenchRecord("gmres", 512, "f64", "b200", 0.02, 5, True, 3e-9, 1.0),
            BenchRecord("lu", 256, "f32", "b200", math.nan, 0, False, math.nan, math.nan)]


def test_csv_round_trip():
    text = emit_report(_recs(), "csv")
    assert text.splitlines()[0] == "method,n,precision,backend,wall_time_s,iterations,converged,relative_residual,speedup"
    back = parse_report_csv(text)
    assert [r.method for r in back] == ["cg", "gmres", "lu"]
    assert back[0].iterations == 12 and back[0].converged is True and math.isnan(back[2].wall_time)


def test_markdown_grid():
    md = emit_report(_recs(), "markdown")
    assert "### f64: speedup vs b200" in md and "| Matrix dimension | cg | gmres |" in md
    assert "| 256 | 1.00x (10 ms) | - |" in md
    assert "### f32: speedup vs b200" in md and "| 256 | - |" in md  # the NaN (failed) point


def test_report_errors():
    with pytest.raises(ValueError):
        emit_report([], "csv")
    with pytest.raises(ValueError):
        emit_report(_recs(), "xml")
    with pytest.raises(ValueError):
        parse_report_csv("a,b\n")


def test_cli_usage_errors(tmp_path, capsys):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%NotMatrixMarket\n")
    assert cli.main(["solve", "--method", "cg", "--matrix", str(bad)]) == 2
    assert "line 1" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["solve", "--method", "jacobi"])
