"""Pin the oracle's BiCGSTAB and Cholesky restatements (oracle/densolve_oracle.py)
to golden vectors produced by the reference itself (tests/golden/make_golden_next.py)."""
import numpy as np
import pytest

from oracle import densolve_oracle as O

BI = ["n64s9", "fixed7", "n17fix6", "n200fix6", "n512s0", "n512s3", "c2_tol8", "f32_n256", "dd_n128"]
CH = ["n16b4", "n64b16", "n200b64", "n256b64", "n256b1", "n96b500", "f32n64", "n1024b64"]


@pytest.mark.parametrize("name", BI)
def test_oracle_bicgstab_matches_reference(golden_next, name):
    kind, n, seed, tol, mi, prec = [str(s) for s in golden_next[f"bi_{name}_spec"]]
    A, b, _ = O.generate_problem(kind, int(n), int(seed), prec)
    x, rep = O.bicgstab(A, b, np.zeros_like(b), float(tol), None if mi == "None" else int(mi))
    assert rep["iterations"] == int(golden_next[f"bi_{name}_iters"])
    assert str(rep["breakdown"]) == str(golden_next[f"bi_{name}_breakdown"])
    np.testing.assert_array_equal(np.array(rep["history"]), golden_next[f"bi_{name}_hist"])
    np.testing.assert_array_equal(x, golden_next[f"bi_{name}_x"])


def test_oracle_bicgstab_kats(golden_next):
    x, rep = O.bicgstab(np.asfortranarray(np.eye(8)), golden_next["bi_eye_b"], np.zeros(8), 1e-4)
    assert rep["iterations"] == int(golden_next["bi_eye_iters"]) == 1
    np.testing.assert_array_equal(x, golden_next["bi_eye_x"])
    A = np.asfortranarray([[0.0, 1.0], [-1.0, 0.0]])
    x, rep = O.bicgstab(A, np.array([1.0, 0.0]), np.zeros(2), 1e-4)
    assert rep["breakdown"] == str(golden_next["bi_rot_breakdown"]) == "rho-breakdown"
    assert rep["iterations"] == int(golden_next["bi_rot_iters"])
    assert len(rep["history"]) == rep["iterations"] + 1


@pytest.mark.parametrize("name", CH)
def test_oracle_cholesky_matches_reference(golden_next, name):
    n, seed, bsz, prec = [str(s) for s in golden_next[f"ch_{name}_spec"]]
    A, b, _ = O.generate_problem("spd", int(n), int(seed), prec)
    L = O.cholesky_factor(A, int(bsz), O.Ops(threads=4))
    if f"ch_{name}_L" in golden_next.files:
        np.testing.assert_array_equal(L, golden_next[f"ch_{name}_L"])
    s = golden_next[f"ch_{name}_Lsum"]
    np.testing.assert_allclose([np.sum(L, dtype=np.float64), np.sum(np.abs(L), dtype=np.float64),
                                np.sum(np.diag(L), dtype=np.float64)], s, rtol=1e-12)
    np.testing.assert_allclose(O.cholesky_solve(L, b), golden_next[f"ch_{name}_x"], rtol=1e-10, atol=1e-12)


def test_oracle_cholesky_notspd_index(golden_next):
    with pytest.raises(O.NotSpd) as e:
        O.cholesky_factor(np.asfortranarray(np.diag([1.0, -1.0])), 2)
    assert e.value.index == int(golden_next["ch_notspd_index"]) == 1
    with pytest.raises(O.NotSpd) as e:
        O.cholesky_factor(golden_next["ch_notspd70_A"], 32)
    assert e.value.index == int(golden_next["ch_notspd70_index"]) == 70
