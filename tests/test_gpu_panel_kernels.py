"""The two LU panel kernels (ds_lu.cu: the CTA-synchronous register-row kernel and the
poller-warp kernel) implement the same panel arithmetic (direct.py:59-79, NumPy
rounding), so the whole blocked factorization must be BITWISE identical whichever
kernel runs each panel.  The kernel choice is read once per process
(DENSOLVE_PANEL_KERNEL: 0 = size-based default, 1 = poller kernel wherever it fits,
2 = CTA-synchronous kernel only), hence one subprocess per setting.  Sizes cover one
CTA (rows <= 224), 2..40 CTAs, more than 40 CTAs, ragged tails, ragged b, fp64 and fp32."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1511_07207_b200 import get_backend, lu_factor_blocked, permutation_matrix

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_1511_07207_b200 import get_backend, lu_factor_blocked
be = get_backend("b200")
for n, b, seed, dt in {cases!r}:
    A = np.asfortranarray(np.random.default_rng(seed).uniform(-1, 1, (n, n)).astype(dt))
    f = lu_factor_blocked(A, b, be)
    h = hashlib.sha256(np.ascontiguousarray(f.packed).tobytes() + np.asarray(f.pivots, np.int64).tobytes())
    print(n, b, h.hexdigest())
"""

CASES = [(200, 64, 1, "float64"), (1000, 48, 2, "float64"), (3000, 64, 3, "float64"), (9000, 64, 4, "float64"),
         (12000, 64, 5, "float64"), (3000, 64, 6, "float32"), (700, 40, 7, "float32")]


def _run(force, cases=CASES, **extra):
    env = dict(os.environ, DENSOLVE_PANEL_KERNEL=str(force), **extra)
    out = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, cases=cases)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return [line.split() for line in out.stdout.strip().splitlines()]


def test_panel_kernels_bitwise_identical():
    runs = {force: _run(force) for force in (0, 1, 2)}
    assert len(runs[0]) == len(CASES)
    assert runs[0] == runs[1] == runs[2]


def test_sm_reservation_is_bitwise_neutral():
    # the tail trailing GEMMs beside the look-ahead panel run as the persistent kernel that
    # leaves the panel's SMs free (ds_blas.cu gemm64_tma_persist_kernel, dynamic tile order):
    # same per-tile DMMA chain, so the same bits as the ordinary launch (DENSOLVE_LU_RESERVE=0)
    cases = [(8192, 64, 8, "float64"), (6000, 64, 9, "float64")]
    on = _run(0, cases)
    off = _run(0, cases, DENSOLVE_LU_RESERVE="0")
    assert len(on) == len(cases) and on == off


def test_u01_fused_is_bitwise_neutral():
    # the outer panel's U01 (TRSM of each 64-row block + the K = 64 update of the rows below)
    # in one launch (ds_blas.cu u01_fused_kernel) vs the TRSM / GEMM launch chain
    cases = [(3000, 64, 10, "float64"), (8192, 64, 11, "float64"), (2048, 64, 12, "float32")]
    on = _run(0, cases)
    off = _run(0, cases, DENSOLVE_LU_U01_FUSED="0")
    assert len(on) == len(cases) and on == off


def test_poller_kernel_factorization_is_valid():
    # the hashes above prove agreement; this checks the shared result is a valid
    # partial-pivoting factorization (in-process, default kernel choice)
    be = get_backend("b200")
    n = 3000
    A = np.asfortranarray(np.random.default_rng(3).uniform(-1, 1, (n, n)))
    f = lu_factor_blocked(A, 64, be)
    L, U = f.lower(), f.upper()
    assert np.max(np.abs(np.tril(f.packed, -1))) <= 1.0
    P = permutation_matrix(f.pivots, n, dtype=np.float64)
    assert np.linalg.norm(P @ A - L @ U) <= 10 * n * np.finfo(np.float64).eps * np.linalg.norm(A)


_ORACLE_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from oracle import densolve_oracle as O
from paper_1511_07207_b200 import get_backend, lu_factor_blocked, lu_factor_unblocked
be = get_backend("b200")
for n, b, seed, dt in {cases!r}:
    A = np.asfortranarray(np.random.default_rng(seed).uniform(-1, 1, (n, n)).astype(dt))
    f = lu_factor_blocked(A, b, be)
    W, piv, _ = O.lu_factor_blocked(A, b)
    same = np.array_equal(np.asarray(f.pivots), piv)
    d = float(np.max(np.abs(f.packed.astype(np.float64) - W.astype(np.float64))))
    fu = lu_factor_unblocked(A, be)
    Wu, pu, _ = O.lu_factor_unblocked(A)
    bit = np.array_equal(np.asarray(fu.pivots), pu) and np.array_equal(fu.packed, Wu)
    print(n, b, int(same), d, int(bit))
"""
ORACLE_CASES = [(200, 64, 11, "float64"), (450, 64, 12, "float64"), (700, 40, 13, "float64"), (300, 32, 14, "float32")]


@pytest.mark.parametrize("force", [1, 2])
def test_each_panel_kernel_matches_the_oracle(force):
    """Each panel kernel, forced everywhere it fits, against the CPU restatement of the
    reference (oracle.lu_factor_blocked, direct.py:50-84): identical pivots, packed factors
    within the blocked-regrouping bound 100 n u max|A|, and the unblocked factorization
    (one panel spanning the matrix, direct.py:25-47) bitwise equal to the oracle's."""
    env = dict(os.environ, DENSOLVE_PANEL_KERNEL=str(force))
    out = subprocess.run([sys.executable, "-c", _ORACLE_SCRIPT.format(root=ROOT, cases=ORACLE_CASES)], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    rows = [line.split() for line in out.stdout.strip().splitlines()]
    assert len(rows) == len(ORACLE_CASES)
    for (n, b, seed, dt), (_, _, same, d, bit) in zip(ORACLE_CASES, rows):
        u = np.finfo(np.dtype(dt)).eps / 2
        assert same == "1", (n, b, "pivots differ from the oracle")
        assert float(d) <= 100 * n * u, (n, b, d)
        assert bit == "1", (n, "unblocked factorization not bitwise equal to the oracle")
