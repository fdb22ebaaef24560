"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU drivers' host
logic: row sharding with padding, rank-ordered reductions, replicated stopping,
the sharded symmetry gate, and the block-cyclic LU with panel broadcast.  The
per-rank compute is the NumPy test double tests/dist_numpy_ops.py; results are
checked against the CPU oracle."""
import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from dist_numpy_ops import NumpyShardOps
        from oracle import densolve_oracle as O
        from paper_1511_07207_b200 import SolverConfig, NotSpdError
        from paper_1511_07207_b200 import distributed as D

        comm, ops = D.TorchComm(), NumpyShardOps()
        out = {}
        if case in ("cg", "cg_pad"):
            n = 64 if case == "cg" else 67
            A, b, _ = O.generate_problem("spd", n, 7)
            n_loc, N = D.row_partition(n, world)
            r0, r1 = rank * n_loc, min(n, (rank + 1) * n_loc)
            A_blk = torch.zeros((n, n_loc), dtype=torch.float64)
            A_blk[:, : r1 - r0] = torch.from_numpy(np.ascontiguousarray(A[r0:r1, :].T))
            b_loc = torch.zeros(n_loc, dtype=torch.float64)
            b_loc[: r1 - r0] = torch.from_numpy(b[r0:r1])
            x, rep = D.cg_solve_sharded(A_blk, b_loc, torch.zeros(n_loc, dtype=torch.float64), n,
                                        SolverConfig(tolerance=1e-10), comm, ops)
            xf = torch.empty(N, dtype=torch.float64)
            comm.allgather(xf, x)
            out = {"x": xf.numpy()[:n].copy(), "it": rep.iterations, "hist": rep.residual_history}
        elif case == "cg_asym":
            A = np.asfortranarray(np.random.default_rng(0).uniform(-1, 1, (8, 8)) + 8 * np.eye(8))
            n_loc, N = D.row_partition(8, world)
            A_blk = torch.from_numpy(np.ascontiguousarray(A[rank * n_loc:(rank + 1) * n_loc, :].T)).clone()
            try:
                D.cg_solve_sharded(A_blk, torch.ones(n_loc, dtype=torch.float64), torch.zeros(n_loc, dtype=torch.float64),
                                   8, SolverConfig(), comm, ops)
                out = {"raised": False}
            except NotSpdError:
                out = {"raised": True}
        elif case.startswith("gmres"):
            orth = "classical" if case.endswith("cgs") else "modified"
            n = 48
            A, b, _ = O.generate_problem("general_nonsymmetric", n, 2)
            n_loc, N = D.row_partition(n, world)
            r0, r1 = rank * n_loc, min(n, (rank + 1) * n_loc)
            A_blk = torch.zeros((n, n_loc), dtype=torch.float64)
            A_blk[:, : r1 - r0] = torch.from_numpy(np.ascontiguousarray(A[r0:r1, :].T))
            b_loc = torch.zeros(n_loc, dtype=torch.float64)
            b_loc[: r1 - r0] = torch.from_numpy(b[r0:r1])
            mi = 7 if case.startswith("gmres_cap") else None
            tol = 1e-300 if mi else 1e-8
            cfg = SolverConfig(tolerance=tol, restart_m=3 if mi else 10, orthogonalization=orth, max_iterations=mi)
            x, rep = D.gmres_solve_sharded(A_blk, b_loc, torch.zeros(n_loc, dtype=torch.float64), n, cfg, comm, ops)
            xf = torch.empty(N, dtype=torch.float64)
            comm.allgather(xf, x)
            out = {"x": xf.numpy()[:n].copy(), "it": rep.iterations, "cycles": rep.restart_cycles,
                   "hist": rep.residual_history, "conv": rep.converged}
        elif case == "lu":
            n, b, NB = 70, 8, 16
            A = np.asfortranarray(np.random.default_rng([0, n, 1]).uniform(-1.0, 1.0, (n, n)))
            W_loc, idx = D.scatter_block_cyclic(A, n, b, rank, world, torch, "cpu", torch.float64, nb_outer=NB)
            piv, sing = D.lu_factor_block_cyclic(W_loc, n, b, comm, ops, nb_outer=NB)
            full = D.gather_block_cyclic(W_loc, idx, n, comm)
            out = {"piv": piv.numpy().copy(), "packed": full, "sing": sing}
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception:
        q.put((rank, {"error": traceback.format_exc()}))


def run_case(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, out = q.get(timeout=240)
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    for r, out in res.items():
        assert "error" not in out, out.get("error")
    return res


@pytest.mark.parametrize("case", ["cg", "cg_pad"])
def test_sharded_cg_matches_oracle(case):
    sys.path.insert(0, ROOT)
    from oracle import densolve_oracle as O
    res = run_case(case)
    n = 64 if case == "cg" else 67
    A, b, _ = O.generate_problem("spd", n, 7)
    xo, ro = O.cg(A, b, np.zeros(n), 1e-10)
    for r in (0, 1):
        assert res[r]["it"] == ro["iterations"]
        np.testing.assert_allclose(res[r]["x"], xo, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(res[r]["hist"], ro["history"], rtol=1e-8)
    # both ranks hold bitwise-identical replicated results
    assert np.array_equal(res[0]["x"], res[1]["x"]) and res[0]["hist"] == res[1]["hist"]


def test_sharded_symmetry_gate():
    res = run_case("cg_asym")
    assert res[0]["raised"] and res[1]["raised"]


@pytest.mark.parametrize("case", ["gmres_mgs", "gmres_cgs", "gmres_cap_cgs"])
def test_sharded_gmres_matches_oracle(case):
    sys.path.insert(0, ROOT)
    from oracle import densolve_oracle as O
    res = run_case(case)
    A, b, _ = O.generate_problem("general_nonsymmetric", 48, 2)
    orth = "classical" if case.endswith("cgs") else "modified"
    if case.startswith("gmres_cap"):
        xo, ro = O.gmres(A, b, np.zeros(48), 1e-300, 3, 7, orth)
    else:
        xo, ro = O.gmres(A, b, np.zeros(48), 1e-8, 10, None, orth)
    for r in (0, 1):
        assert abs(res[r]["it"] - ro["iterations"]) <= 1
        assert res[r]["conv"] == ro["converged"]
        if ro["converged"]:
            np.testing.assert_allclose(res[r]["x"], xo, rtol=1e-6, atol=1e-9)
    assert res[0]["cycles"] == res[1]["cycles"] and res[0]["hist"] == res[1]["hist"]
    if case.startswith("gmres_cap"):
        assert res[0]["cycles"] == ro["cycles"] == [0, 3, 6]


def test_block_cyclic_lu_matches_oracle():
    sys.path.insert(0, ROOT)
    from oracle import densolve_oracle as O
    res = run_case("lu")
    n, b = 70, 8
    A = np.asfortranarray(np.random.default_rng([0, n, 1]).uniform(-1.0, 1.0, (n, n)))
    W, piv, _ = O.lu_factor_blocked(A, b)
    for r in (0, 1):
        assert np.array_equal(res[r]["piv"], piv)
        np.testing.assert_allclose(res[r]["packed"], W, rtol=0, atol=1e-11)
        assert not res[r]["sing"]


def test_partition_helpers():
    sys.path.insert(0, ROOT)
    from paper_1511_07207_b200 import distributed as D
    assert D.row_partition(10, 4) == (3, 12)
    assert D.row_partition(32768, 8) == (4096, 32768)
    assert [D.block_owner(k, 3) for k in range(7)] == [0, 1, 2, 0, 1, 2, 0]
    assert D.local_blocks(7, 1, 3) == [1, 4]
    assert D.outer_block(64, 32768) == 256 and D.outer_block(64, 100) == 100 and D.outer_block(300, 1000) == 300
    parts = np.array([4.0, 2.0, 1.0, 9.0, 3.0, 1.0])  # ||(2)||, ||(3)||
    s2, nrm = D.combine3_host(parts)
    assert s2 == 13.0 and abs(nrm - np.sqrt(13.0)) < 1e-15
