"""GPU tests of the sweep and CLI plumbing over the b200 backend (test_harness.py:132-200,
test_cli.py patterns) and of Matrix Market input feeding a device solve."""
import os

import numpy as np
import pytest

from paper_1511_07207_b200 import SolverConfig, cli, read_matrix_market, relative_residual, solve_system
from paper_1511_07207_b200.harness import emit_report, parse_report_csv, run_benchmark

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_single_record_speedup_one():
    recs = run_benchmark(["cg"], [128], ["f64"], ["b200"], SolverConfig(tolerance=1e-8), repeats=1)
    assert len(recs) == 1 and recs[0].speedup_vs_reference == 1.0 and recs[0].converged


def test_sweep_shape_and_reports():
    methods = ["cg", "gmres", "bicgstab", "lu-blocked", "cholesky"]
    recs = run_benchmark(methods, [64, 128], ["f64"], ["b200"], SolverConfig(tolerance=1e-8), repeats=1)
    assert len(recs) == len(methods) * 2
    assert all(r.converged for r in recs)
    assert all(r.relative_residual <= 1e-7 for r in recs)
    back = parse_report_csv(emit_report(recs, "csv"))
    assert [(r.method, r.n) for r in back] == [(r.method, r.n) for r in recs]
    md = emit_report(recs, "markdown")
    assert "| Matrix dimension | cg | gmres | bicgstab |" in md


def test_nonconverged_solve_recorded():
    # a capped, non-converged solve is a record (converged=False), not an exception
    recs = run_benchmark(["cg"], [32], ["f64"], ["b200"], SolverConfig(tolerance=1e-8, max_iterations=1),
                         repeats=1)
    assert len(recs) == 1 and not recs[0].converged


def test_empty_inputs_rejected():
    with pytest.raises(ValueError):
        run_benchmark([], [64], ["f64"], ["b200"], SolverConfig())
    with pytest.raises(NotImplementedError):
        run_benchmark(["jacobi"], [64], ["f64"], ["b200"], SolverConfig())


def test_matrix_market_system_solves(tmp_path):
    rng = np.random.default_rng(9)
    M = rng.uniform(-1, 1, (40, 40))
    S = M @ M.T + 40 * np.eye(40)
    p = tmp_path / "spd.mtx"
    with open(p, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real symmetric\n" + f"40 40 {40 * 41 // 2}\n")
        for j in range(40):
            for i in range(j, 40):
                fh.write(f"{i + 1} {j + 1} {float(S[i, j])!r}\n")
    A = read_matrix_market(p)
    b = A @ np.ones(40)
    for method in ("cg", "cholesky", "lu-blocked", "gmres", "bicgstab"):
        x, rep = solve_system(method, A, b, None, SolverConfig(tolerance=1e-10), "b200")
        assert relative_residual(A, x, b) <= 1e-9, method


def test_cli_solve_and_bench(tmp_path, capsys):
    assert cli.main(["solve", "--method", "cg", "--n", "64", "--tol", "1e-8"]) == 0
    assert "converged" in capsys.readouterr().out
    out = tmp_path / "r.csv"
    assert cli.main(["bench", "--method", "cg,lu", "--sizes", "32,64", "--output", "csv", "--out", str(out),
                     "--repeats", "1"]) == 0
    assert len(parse_report_csv(out.read_text())) == 4
    mtx = os.path.join(HERE, "golden", "mtx", "coord_diag.mtx")
    assert cli.main(["solve", "--method", "lu", "--matrix", mtx]) == 0


def test_sweep_against_the_reference_backend():
    """b200 beside the unmodified reference's CPU backend in one sweep (baseline/_ref): the
    speedup column is relative to the first backend, and both solve the same system."""
    import sys
    ref = os.path.join(os.path.dirname(HERE), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "densolve")):
        pytest.skip("baseline/_ref not installed")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    recs = run_benchmark(["cg", "lu-blocked"], [512], ["f64"], ["reference", "b200"],
                         SolverConfig(tolerance=1e-8), repeats=1)
    assert [(r.method, r.backend) for r in recs] == [("cg", "reference"), ("cg", "b200"),
                                                     ("lu-blocked", "reference"), ("lu-blocked", "b200")]
    assert all(r.converged for r in recs)
    assert recs[0].iterations == recs[1].iterations
    assert recs[0].speedup_vs_reference == 1.0 and recs[1].speedup_vs_reference > 1.0
