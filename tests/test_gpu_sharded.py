"""Row-sharded CG behind the reference API (get_backend("b200", devices=[...]) and
get_backend("b200", distributed=True)) against the CPU oracle (krylov.py:36-72).

The test box has one GPU, so several shards share it: devices=[0, 0] runs two shards
with their own streams and exchange regions on GPU 0 (the P2P stores are then local
stores, the flag protocol and the all-gather fusion are exercised unchanged), and the
distributed test runs two processes on GPU 0 that map each other's exchange regions
through CUDA IPC."""
import os
import sys
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle import densolve_oracle as O  # noqa: E402


def _spd(n, seed):
    A, b, _ = O.generate_problem("spd", n, seed)
    return A, b


@pytest.mark.parametrize("devices,n", [([0], 300), ([0, 0], 300), ([0, 0, 0], 301), ([0, 0, 0, 0], 257)])
def test_sharded_cg_matches_oracle(devices, n):
    from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend

    A, b = _spd(n, 7)
    be = get_backend("b200", devices=devices)
    x, rep = cg_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10), be)
    xo, ro = O.cg(A, b, np.zeros_like(b), 1e-10)
    assert rep.converged
    assert abs(rep.iterations - ro["iterations"]) <= 1
    k = min(len(rep.residual_history), len(ro["history"]))
    np.testing.assert_allclose(rep.residual_history[:k], ro["history"][:k], rtol=1e-6)
    assert np.linalg.norm(x - xo, np.inf) <= 1e-9 * np.linalg.norm(xo, np.inf)
    # the reference's counter law (one gemv per iteration + setup)
    assert be.counters.gemv_calls == rep.iterations + 1


def test_sharded_cg_equals_across_shard_counts():
    """The shard-ordered record combination is deterministic: repeated solves are bitwise
    equal, and every shard count converges to the same solution."""
    from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend

    A, b = _spd(512, 3)
    cfg = SolverConfig(tolerance=1e-12)
    be2 = get_backend("b200", devices=[0, 0])
    x1, r1 = cg_solve(A, b, np.zeros_like(b), cfg, be2)
    x2, r2 = cg_solve(A, b, np.zeros_like(b), cfg, be2)
    assert np.array_equal(x1, x2) and r1.residual_history == r2.residual_history
    x0_, r0_ = cg_solve(A, b, np.zeros_like(b), cfg, get_backend("b200"))
    assert abs(r1.iterations - r0_.iterations) <= 1
    assert np.linalg.norm(x1 - x0_, np.inf) <= 1e-10 * np.linalg.norm(x0_, np.inf)


def test_sharded_cg_fp32_and_c_order():
    from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend

    A, b = _spd(200, 5)
    A32, b32 = np.ascontiguousarray(A.astype(np.float32)), b.astype(np.float32)
    x, rep = cg_solve(A32, b32, np.zeros_like(b32), SolverConfig(tolerance=1e-5), get_backend("b200", devices=[0, 0]))
    xo, ro = O.cg(np.asfortranarray(A32), b32, np.zeros_like(b32), 1e-5)
    assert x.dtype == np.float32 and rep.converged
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert np.linalg.norm(x - xo, np.inf) <= 1e-3 * np.linalg.norm(xo, np.inf)


def test_sharded_cg_nonzero_x0_and_device_resident():
    from paper_1511_07207_b200 import SolverConfig, ShardedVector, cg_solve, get_backend

    A, b = _spd(333, 11)
    x0 = np.random.default_rng(1).standard_normal(333)
    be = get_backend("b200", devices=[0, 0, 0])
    dA, db, dx0 = be.stage_in(A, b, x0)
    x, rep = cg_solve(dA, db, dx0, SolverConfig(tolerance=1e-10), be)
    assert isinstance(x, ShardedVector)
    xh = be.stage_out(x)
    xo, ro = O.cg(A, b, x0, 1e-10)
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert np.linalg.norm(xh - xo, np.inf) <= 1e-9 * np.linalg.norm(xo, np.inf)


def test_sharded_cg_errors():
    from paper_1511_07207_b200 import (DegenerateRhsError, NotSpdError, SolverConfig, cg_solve, get_backend)

    be = get_backend("b200", devices=[0, 0])
    A, b = _spd(128, 2)
    B = A.copy(order="F")
    B[3, 100] += 1e-3  # not symmetric: caught by the sharded gate (off-diagonal block pair)
    with pytest.raises(NotSpdError):
        cg_solve(B, b, np.zeros_like(b), SolverConfig(tolerance=1e-8), be)
    with pytest.raises(NotSpdError):  # symmetric, negative definite: p'Ap <= 0
        cg_solve(np.asfortranarray(-A), b, np.zeros_like(b), SolverConfig(tolerance=1e-8), be)
    with pytest.raises(DegenerateRhsError):
        cg_solve(A, np.zeros_like(b), np.zeros_like(b), SolverConfig(tolerance=1e-8), be)
    # the shard set is still usable after the errors
    x, rep = cg_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-8), be)
    assert rep.converged


def _dist_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK="0")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend

        A, b = _spd(301, 9)  # same host arrays on every rank (the reference call)
        be = get_backend("b200", distributed=True, device=0)
        x, rep = cg_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10), be)
        from paper_1511_07207_b200 import gmres_solve
        An, bn, _ = O.generate_problem("general_nonsymmetric", 301, 4)
        xg, repg = gmres_solve(An, bn, np.zeros_like(bn), SolverConfig(tolerance=1e-10, restart_m=8), be)
        from paper_1511_07207_b200 import lu_factor_blocked
        Au = np.asfortranarray(np.random.default_rng(600).uniform(-1, 1, (600, 600)))
        f = lu_factor_blocked(Au, 64, be)
        q.put((rank, x, rep.iterations, rep.residual_history, xg, (repg.iterations, np.asarray(f.pivots), f.packed)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        q.put((rank, traceback.format_exc(), None, None, None, None))


def test_distributed_cg_two_processes_ipc():
    import torch.multiprocessing as mp

    from test_distributed_gloo import _free_port

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(60)
    for r, x, it, h, _, _ in res:
        assert it is not None, x
    A, b = _spd(301, 9)
    xo, ro = O.cg(A, b, np.zeros_like(b), 1e-10)
    (_, xa, ia, ha, ga, gia), (_, xb, ib, hb, gb, gib) = sorted(res, key=lambda t: t[0])
    assert ia == ib and ha == hb and np.array_equal(xa, xb)  # replicated decisions
    assert abs(ia - ro["iterations"]) <= 1
    assert np.linalg.norm(xa - xo, np.inf) <= 1e-9 * np.linalg.norm(xo, np.inf)
    An, bn, _ = O.generate_problem("general_nonsymmetric", 301, 4)
    xgo, rgo = O.gmres(An, bn, np.zeros_like(bn), 1e-10, 8)
    (gia, pa, La), (gib, pb, Lb) = gia, gib
    assert gia == gib and np.array_equal(ga, gb)
    assert abs(gia - rgo["iterations"]) <= 1
    assert np.linalg.norm(ga - xgo, np.inf) <= 1e-8 * np.linalg.norm(xgo, np.inf)
    # block-cyclic LU over the two processes: identical factors on both ranks, the oracle's pivots
    Au = np.asfortranarray(np.random.default_rng(600).uniform(-1, 1, (600, 600)))
    W, piv, _ = O.lu_factor_blocked(Au, 64)
    assert np.array_equal(pa, pb) and np.array_equal(La, Lb)
    assert np.array_equal(pa, piv)
    assert np.abs(La - W).max() <= 100 * 600 * np.finfo(np.float64).eps


@pytest.mark.parametrize("devices,m,orth", [([0], 20, "modified"), ([0, 0], 20, "modified"),
                                            ([0, 0, 0], 5, "modified"), ([0, 0], 7, "classical")])
def test_sharded_gmres_matches_oracle(devices, m, orth):
    """krylov.gmres_solve with A split by rows: ds_gmres_sharded (the Arnoldi loop in the
    library, records all-gathered over peer memory) against the oracle, restarts included."""
    from paper_1511_07207_b200 import SolverConfig, get_backend, gmres_solve

    A, b, _ = O.generate_problem("general_nonsymmetric", 301, 4)
    be = get_backend("b200", devices=devices)
    cfg = SolverConfig(tolerance=1e-10, restart_m=m, orthogonalization=orth)
    x, rep = gmres_solve(A, b, np.zeros_like(b), cfg, be)
    xo, ro = O.gmres(A, b, np.zeros_like(b), 1e-10, m, orth=orth)
    assert rep.converged and ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    k = min(len(rep.residual_history), len(ro["history"])) - 1
    np.testing.assert_allclose(rep.residual_history[:k], ro["history"][:k], rtol=1e-6)
    if rep.iterations == ro["iterations"]:
        assert rep.restart_cycles == ro["cycles"]
    assert np.linalg.norm(x - xo, np.inf) <= 1e-8 * np.linalg.norm(xo, np.inf)
    # the single-GPU solver agrees too
    x1, rep1 = gmres_solve(A, b, np.zeros_like(b), cfg, get_backend("b200"))
    assert abs(rep.iterations - rep1.iterations) <= 1


def test_sharded_gmres_fp32_and_errors():
    from paper_1511_07207_b200 import DegenerateRhsError, SolverConfig, get_backend, gmres_solve

    A, b, _ = O.generate_problem("general_nonsymmetric", 200, 6)
    A32, b32 = np.asfortranarray(A.astype(np.float32)), b.astype(np.float32)
    be = get_backend("b200", devices=[0, 0])
    x, rep = gmres_solve(A32, b32, np.zeros_like(b32), SolverConfig(tolerance=1e-5, restart_m=30), be)
    xo, ro = O.gmres(A32, b32, np.zeros_like(b32), 1e-5, 30)
    assert x.dtype == np.float32 and rep.converged
    assert abs(rep.iterations - ro["iterations"]) <= 1
    with pytest.raises(DegenerateRhsError):
        gmres_solve(A, np.zeros_like(b), np.zeros_like(b), SolverConfig(tolerance=1e-8), be)
    with pytest.raises(ValueError):
        gmres_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-8, restart_m=64), be)
    # one shard: the fused single-GPU step, no restart limit
    x1, r1 = gmres_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-8, restart_m=80),
                         get_backend("b200", devices=[0]))
    assert r1.converged


@pytest.mark.parametrize("devices,n,b", [([0], 300, 64), ([0, 0], 600, 64), ([0, 0, 0], 777, 32),
                                         ([0, 0], 1100, 64), ([0, 0, 0, 0], 2100, 48)])
def test_sharded_lu_matches_oracle(devices, n, b):
    """direct.lu_factor_blocked with the columns dealt block-cyclically to the shards
    (ds_lu_block_cyclic: panels broadcast over peer memory, look-ahead): the pivot sequence
    equals the oracle's, the factors agree within the blocked-vs-unblocked bound, lu_solve
    solves."""
    from paper_1511_07207_b200 import get_backend, lu_factor_blocked, lu_solve

    A = np.asfortranarray(np.random.default_rng(n).uniform(-1, 1, (n, n)))
    be = get_backend("b200", devices=devices)
    f = lu_factor_blocked(A, b, be)
    W, piv, _ = O.lu_factor_blocked(A, b)
    assert np.array_equal(np.asarray(f.pivots), piv)
    assert np.abs(f.packed - W).max() <= 100 * n * np.finfo(np.float64).eps * np.abs(A).max()
    rhs = np.ones(n)
    x = lu_solve(f, rhs)
    assert np.linalg.norm(A @ x - rhs) <= 1e-10 * np.linalg.norm(A, 1) * np.linalg.norm(x)


def test_sharded_edge_cases():
    """Edge cases through the sharded engines (2 shards): CG from the exact solution (0
    iterations), GMRES happy breakdown on the identity, a singular block-cyclic LU, fp32
    block-cyclic LU against the oracle."""
    from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend, gmres_solve, lu_factor_blocked

    be = get_backend("b200", devices=[0, 0])
    A, b = _spd(160, 21)
    xs = np.linalg.solve(A, b)
    x, rep = cg_solve(A, b, xs, SolverConfig(tolerance=1e-8), be)
    xo, ro = O.cg(A, b, xs, 1e-8)
    assert rep.iterations == ro["iterations"] and rep.converged
    I = np.asfortranarray(np.eye(90))
    bi = np.random.default_rng(3).standard_normal(90)
    xg, rg = gmres_solve(I, bi, np.zeros(90), SolverConfig(tolerance=1e-10, restart_m=10), be)
    xgo, rgo = O.gmres(I, bi, np.zeros(90), 1e-10, 10)
    assert rg.converged and rg.iterations == rgo["iterations"] and rg.breakdown == rgo["breakdown"]
    assert np.allclose(xg, bi)
    S = np.asfortranarray(np.random.default_rng(4).uniform(-1, 1, (700, 700)))
    S[:, 400] = 0.0
    f = lu_factor_blocked(S, 64, be)
    W, piv, sing = O.lu_factor_blocked(S, 64)
    assert f.singular == bool(sing) and np.array_equal(np.asarray(f.pivots), piv)
    A32 = np.asfortranarray(np.random.default_rng(5).uniform(-1, 1, (520, 520)).astype(np.float32))
    f32 = lu_factor_blocked(A32, 32, be)
    W32, piv32, _ = O.lu_factor_blocked(A32, 32)
    assert f32.packed.dtype == np.float32 and np.array_equal(np.asarray(f32.pivots), piv32)
    assert np.abs(f32.packed - W32).max() <= 100 * 520 * np.finfo(np.float32).eps
