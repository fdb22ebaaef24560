"""CPU-side checks of the drop-in boundary (no GPU needed): the C-ABI library loads
and exports every symbol include/densolve_b200.h declares; the ctypes binding
types all of them; the product package never imports the oracle and has no CPU
fallback; validation happens on the host before any device work."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "densolve_b200.h")
LIB = os.path.join(ROOT, "paper_1511_07207_b200", "libdensolve_b200.so")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|const char\*)\s+(ds_\w+)\s*\(", text)))


def test_header_declares_the_reference_entry_points():
    syms = header_symbols()
    for s in ["ds_cg", "ds_gmres", "ds_lu_factor", "ds_lu_solve", "ds_forward_substitution",
              "ds_backward_substitution", "ds_gemv", "ds_dot", "ds_nrm2", "ds_axpy", "ds_scal", "ds_iamax",
              "ds_ger", "ds_gemm", "ds_trsm_lower_unit", "ds_trsm_upper", "ds_upload_matrix",
              "ds_cg_shard_update", "ds_lu_panel", "ds_laswp"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build the library first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (ds_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for s in header_symbols():
        assert hasattr(lib, s)


def test_ctypes_binding_covers_the_header():
    from paper_1511_07207_b200 import _lib
    assert sorted(_lib.EXPORTED_SYMBOLS) == header_symbols()
    lib = _lib.load_library()
    assert lib.ds_version().decode().startswith("densolve_b200")


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_sass_uses_dmma_for_fp64_gemm():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = out.split("Function : ")
    gemm = [f for f in funcs if "gemm64_kernel" in f.split("\n", 1)[0]]
    assert gemm and all("DMMA.8x8x4" in f for f in gemm)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1511_07207_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", src).replace("oracle/", ""), f


def test_no_cpu_fallback_without_gpu():
    from paper_1511_07207_b200 import SolverConfig, _lib, cg_solve
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError):
        cg_solve(np.eye(3), np.ones(3), np.zeros(3), SolverConfig(), "b200")


def test_validation_before_device_work():
    from paper_1511_07207_b200 import (DimensionError, PrecisionError, SolverConfig, cg_solve, gmres_solve,
                                       lu_factor_blocked, lu_solve, LuFactors, SingularMatrixError)
    with pytest.raises(DimensionError):
        cg_solve(np.eye(3), np.ones(2), np.zeros(3), SolverConfig(), "b200")
    with pytest.raises(PrecisionError):
        gmres_solve(np.eye(3, dtype=np.float32), np.ones(3), np.zeros(3), SolverConfig(), "b200")
    with pytest.raises(DimensionError):
        lu_factor_blocked(np.ones((3, 4)), 2, "b200")
    with pytest.raises(SingularMatrixError):
        lu_solve(LuFactors(packed=np.eye(2), pivots=np.array([0, 1]), singular=True), np.ones(2))
    with pytest.raises(DimensionError):
        lu_solve(LuFactors(packed=np.eye(2), pivots=np.array([0, 1])), np.ones(3))


def test_reference_types_and_config():
    from paper_1511_07207_b200 import (BackendCounters, SolverConfig, apply_pivots, apply_pivots_inverse,
                                       get_backend, permutation_matrix, permutation_sign)
    cfg = SolverConfig()
    assert (cfg.tolerance, cfg.restart_m, cfg.block_size_b, cfg.orthogonalization) == (1e-4, 35, 64, "modified")
    assert cfg.iteration_cap(50) == 500 and SolverConfig(max_iterations=7).iteration_cap(50) == 7
    for kw in [{"tolerance": 0.0}, {"restart_m": 0}, {"block_size_b": 0}, {"orthogonalization": "none"},
               {"max_iterations": 0}]:
        with pytest.raises(ValueError):
            SolverConfig(**kw)
    rng = np.random.default_rng(0)
    piv = np.array([rng.integers(k, 17) for k in range(17)])
    v = rng.standard_normal(17)
    assert np.array_equal(apply_pivots_inverse(piv, apply_pivots(piv, v)), v)
    assert np.array_equal(permutation_matrix(np.array([1, 1]), 2), [[0.0, 1.0], [1.0, 0.0]])
    assert permutation_sign(np.array([1, 1])) == -1
    c = BackendCounters()
    c.dot_calls, c.dot_flops = 3, 6.0
    assert c.total_calls() == 3 and c.snapshot().dot_flops == 6.0
    c.reset()
    assert c.total_calls() == 0
    assert get_backend("b200").name == "b200"
    with pytest.raises(ValueError):
        get_backend("gpu")
