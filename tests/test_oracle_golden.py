"""Pin the CPU oracle (oracle/densolve_oracle.py) to golden vectors produced by
the reference implementation itself (tests/golden/make_golden.py)."""
import hashlib

import numpy as np
import pytest

from oracle import densolve_oracle as O
from paper_1511_07207_b200 import harness as H


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asfortranarray(a)).tobytes(order="F")).hexdigest()


def test_generators_bitwise_match_reference(golden):
    for i in range(int(golden["gen_count"])):
        kind, n, seed, prec = [str(s) for s in golden[f"gen{i}_spec"]]
        A, b, _ = O.generate_problem(kind, int(n), int(seed), prec)
        assert sha(A) == str(golden[f"gen{i}_shaA"]), (kind, n, seed, prec)
        assert sha(b) == str(golden[f"gen{i}_shab"])
        # the package's own generator (used by bench/tests on the GPU box) is bit-identical too
        A2, b2, _ = H.generate_problem(H.ProblemSpec(kind=kind, n=int(n), seed=int(seed), precision=prec))
        assert sha(A2) == str(golden[f"gen{i}_shaA"])
        assert sha(b2) == str(golden[f"gen{i}_shab"])
    for i in range(3):
        n, seed = (int(v) for v in golden[f"ws{i}_spec"])
        assert sha(O.generate_well_separated(n, seed)) == str(golden[f"ws{i}_sha"])
        assert sha(H.generate_well_separated(n, seed)) == str(golden[f"ws{i}_sha"])


@pytest.mark.parametrize("name", ["c1s0", "c1s1", "c1s2", "n64s7", "fixed", "f32"])
def test_oracle_cg_matches_reference(golden, name):
    kind, n, seed, prec, tol, mi = [str(s) for s in golden[f"cg_{name}_spec"]]
    A, b, _ = O.generate_problem(kind, int(n), int(seed), prec)
    x, rep = O.cg(A, b, np.zeros_like(b), float(tol), None if mi == "None" else int(mi))
    assert rep["iterations"] == int(golden[f"cg_{name}_iters"])
    np.testing.assert_allclose(rep["history"], golden[f"cg_{name}_hist"], rtol=1e-9)
    np.testing.assert_allclose(x, golden[f"cg_{name}_x"], rtol=1e-9, atol=1e-12)


def test_oracle_cg_k_eigen(golden):
    for k in (1, 3, 5):
        for seed in range(3):
            x, rep = O.cg(golden[f"cgk{k}_{seed}_A"], golden[f"cgk{k}_{seed}_b"], np.zeros(64), 1e-10)
            assert rep["iterations"] == int(golden[f"cgk{k}_{seed}_iters"]) <= k + 2


GM = ["n48s2_mgs", "n48s2_cgs", "n128s8_r20", "n64s4_r5", "n64s4_r5_cgs", "c2_tol4", "c2_tol8",
      "c2_fixed", "n512s0_r35", "f32_n256", "cap7"]


@pytest.mark.parametrize("name", GM)
def test_oracle_gmres_matches_reference(golden, name):
    n, seed, tol, m, orth, mi, prec = [str(s) for s in golden[f"gm_{name}_spec"]]
    A, b, _ = O.generate_problem("general_nonsymmetric", int(n), int(seed), prec)
    x, rep = O.gmres(A, b, np.zeros_like(b), float(tol), int(m), None if mi == "None" else int(mi), orth)
    assert rep["iterations"] == int(golden[f"gm_{name}_iters"])
    assert rep["cycles"] == list(golden[f"gm_{name}_cycles"])
    assert rep["converged"] == bool(golden[f"gm_{name}_conv"])
    np.testing.assert_allclose(rep["history"], golden[f"gm_{name}_hist"], rtol=1e-6)
    np.testing.assert_allclose(x, golden[f"gm_{name}_x"], rtol=1e-6, atol=1e-9)


def test_oracle_gmres_rotation(golden):
    A = np.asfortranarray([[0.0, 1.0], [-1.0, 0.0]])
    x, rep = O.gmres(A, np.array([1.0, 0.0]), np.zeros(2), 1e-12)
    assert rep["iterations"] == int(golden["gm_rot_iters"]) == 2
    np.testing.assert_allclose(x, golden["gm_rot_x"], atol=1e-12)


def test_oracle_lu_bitwise(golden):
    A = O.generate_well_separated(64, 3)
    W, piv, s = O.lu_factor_unblocked(A)
    assert np.array_equal(piv, golden["lu_ws64_unb_piv"])
    assert np.array_equal(W, golden["lu_ws64_unb_packed"])
    for b in (1, 8, 32, 64):
        W, piv, _ = O.lu_factor_blocked(A, b)
        assert np.array_equal(piv, golden[f"lu_ws64_b{b}_piv"])
        np.testing.assert_allclose(W, golden[f"lu_ws64_b{b}_packed"], rtol=0, atol=1e-12)
    U = golden["lu_u128_A"]
    for b in (8, 32):
        W, piv, _ = O.lu_factor_blocked(U, b)
        assert np.array_equal(piv, golden[f"lu_u128_b{b}_piv"])
        np.testing.assert_allclose(W, golden[f"lu_u128_b{b}_packed"], rtol=0, atol=1e-12)
    W, piv, _ = O.lu_factor_unblocked(U)
    assert np.array_equal(piv, golden["lu_u128_unb_piv"])
    assert np.array_equal(W, golden["lu_u128_unb_packed"])
    W, piv, _ = O.lu_factor_unblocked(np.asfortranarray([[4.0, 3.0], [6.0, 3.0]]))
    assert np.array_equal(W, golden["lu_kat2_packed"]) and list(piv) == [1, 1]


@pytest.mark.parametrize("n", [512, 1024])
def test_oracle_lu_harness_family(golden, n):
    A, b, _ = O.generate_problem("general_nonsymmetric", n, 0)
    W, piv, _ = O.lu_factor_blocked(A, 64)
    assert np.array_equal(piv, golden[f"lu_gn{n}_piv"])
    assert np.array_equal(piv, np.arange(n))  # diagonally dominant: no swaps
    np.testing.assert_allclose(O.lu_solve(W, piv, b), golden[f"lu_gn{n}_x"], rtol=1e-12)


@pytest.mark.parametrize("n", [256, 512])
def test_oracle_lu_uniform_family(golden, n):
    A = np.asfortranarray(np.random.default_rng([0, n, 1]).uniform(-1.0, 1.0, (n, n)))
    b = np.random.default_rng([0, n, 2]).uniform(-1.0, 1.0, n)
    W, piv, _ = O.lu_factor_blocked(A, 64)
    assert np.array_equal(piv, golden[f"lu_uni{n}_piv"])
    np.testing.assert_allclose(O.lu_solve(W, piv, b), golden[f"lu_uni{n}_x"], rtol=1e-10)


def test_oracle_lu_f32(golden):
    W, piv, _ = O.lu_factor_blocked(golden["lu_f32_64_A"], 64)
    assert np.array_equal(piv, golden["lu_f32_64_piv"])
    assert np.array_equal(W, golden["lu_f32_64_packed"])


def test_oracle_level1_semantics(golden):
    ops = O.Ops()
    assert ops.nrm2(np.array([1e300, 1e300])) == float(golden["nrm2_big"])
    assert ops.nrm2(np.array([3.0, 4.0])) == float(golden["nrm2_34"])
    assert ops.iamax(np.array([2.0, -2.0])) == int(golden["iamax_tie"]) == 0
