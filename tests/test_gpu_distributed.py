"""The multi-GPU drivers with the REAL device kernels (CudaShardOps -> C ABI):
two ranks share the one GPU of the test box; collectives are staged through
host memory over gloo (NCCL refuses two ranks on one device).  Checks the
sharded CG / GMRES / block-cyclic LU against the CPU oracle."""
import os
import sys
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_distributed_gloo import _free_port  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class StagedComm:
    """gloo collectives on CUDA tensors via host staging (test infrastructure)."""

    def __init__(self):
        self.rank, self.size = dist.get_rank(), dist.get_world_size()

    def allgather(self, out, inp):
        o = out.detach().cpu()
        dist.all_gather_into_tensor(o, inp.detach().contiguous().cpu())
        out.copy_(o)

    def broadcast(self, t, src):
        h = t.detach().cpu()
        dist.broadcast(h, src)
        t.copy_(h)

    def allreduce_max(self, t):
        h = t.detach().cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        t.copy_(h)

    def alltoall(self, out, inp):
        o = out.detach().cpu()
        dist.all_to_all_single(o, inp.detach().contiguous().cpu())
        out.copy_(o)

    def barrier(self):
        dist.barrier()


def _worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from oracle import densolve_oracle as O
        from paper_1511_07207_b200 import SolverConfig, get_backend
        from paper_1511_07207_b200 import distributed as D

        be = get_backend("b200", device=0)
        ops = D.CudaShardOps(be.ctx)
        ops.bind_current_stream()
        comm = StagedComm()
        dev = "cuda"
        out = {}
        if case == "cg":
            n = 300
            A, b, _ = O.generate_problem("spd", n, 3)
            n_loc, N = D.row_partition(n, world)
            r0, r1 = rank * n_loc, min(n, (rank + 1) * n_loc)
            A_blk = torch.zeros((n, n_loc), dtype=torch.float64, device=dev)
            A_blk[:, : r1 - r0] = torch.from_numpy(np.ascontiguousarray(A[r0:r1, :].T)).to(dev)
            b_loc = torch.zeros(n_loc, dtype=torch.float64, device=dev)
            b_loc[: r1 - r0] = torch.from_numpy(b[r0:r1]).to(dev)
            x, rep = D.cg_solve_sharded(A_blk, b_loc, torch.zeros(n_loc, dtype=torch.float64, device=dev), n,
                                        SolverConfig(tolerance=1e-10), comm, ops)
            xf = torch.empty(N, dtype=torch.float64, device=dev)
            comm.allgather(xf, x)
            out = {"x": xf.cpu().numpy()[:n].copy(), "it": rep.iterations, "hist": rep.residual_history}
        elif case in ("gmres", "gmres_cgs"):
            n = 200
            A, b, _ = O.generate_problem("general_nonsymmetric", n, 1)
            n_loc, N = D.row_partition(n, world)
            r0, r1 = rank * n_loc, min(n, (rank + 1) * n_loc)
            A_blk = torch.zeros((n, n_loc), dtype=torch.float64, device=dev)
            A_blk[:, : r1 - r0] = torch.from_numpy(np.ascontiguousarray(A[r0:r1, :].T)).to(dev)
            b_loc = torch.zeros(n_loc, dtype=torch.float64, device=dev)
            b_loc[: r1 - r0] = torch.from_numpy(b[r0:r1]).to(dev)
            orth = "classical" if case == "gmres_cgs" else "modified"
            cfg = SolverConfig(tolerance=1e-10, restart_m=4, orthogonalization=orth)
            x, rep = D.gmres_solve_sharded(A_blk, b_loc, torch.zeros(n_loc, dtype=torch.float64, device=dev), n,
                                           cfg, comm, ops)
            xf = torch.empty(N, dtype=torch.float64, device=dev)
            comm.allgather(xf, x)
            out = {"x": xf.cpu().numpy()[:n].copy(), "it": rep.iterations, "cycles": rep.restart_cycles,
                   "conv": rep.converged}
        elif case == "lu":
            n, b, NB = 300, 16, 64
            A = np.asfortranarray(np.random.default_rng([0, n, 1]).uniform(-1.0, 1.0, (n, n)))
            W_loc, idx = D.scatter_block_cyclic(A, n, b, rank, world, torch, dev, torch.float64, nb_outer=NB)
            piv, sing = D.lu_factor_block_cyclic(W_loc, n, b, comm, ops, nb_outer=NB)
            full = D.gather_block_cyclic(W_loc, idx, n, comm)
            out = {"piv": piv.cpu().numpy().copy(), "packed": full}
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
        r, out = q.get(timeout=300)
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    for out in res.values():
        assert "error" not in out, out.get("error")
    return res


def test_sharded_cg_device_kernels():
    from oracle import densolve_oracle as O
    res = run_case("cg")
    A, b, _ = O.generate_problem("spd", 300, 3)
    xo, ro = O.cg(A, b, np.zeros(300), 1e-10)
    for r in (0, 1):
        assert abs(res[r]["it"] - ro["iterations"]) <= 1
        assert np.linalg.norm(res[r]["x"] - xo, np.inf) <= 1e-9 * np.linalg.norm(xo, np.inf)
    assert np.array_equal(res[0]["x"], res[1]["x"]) and res[0]["hist"] == res[1]["hist"]


@pytest.mark.parametrize("case", ["gmres", "gmres_cgs"])
def test_sharded_gmres_device_kernels(case):
    from oracle import densolve_oracle as O
    res = run_case(case)
    A, b, _ = O.generate_problem("general_nonsymmetric", 200, 1)
    orth = "classical" if case == "gmres_cgs" else "modified"
    xo, ro = O.gmres(A, b, np.zeros(200), 1e-10, 4, None, orth)
    for r in (0, 1):
        assert res[r]["conv"] and abs(res[r]["it"] - ro["iterations"]) <= 1
        assert np.linalg.norm(res[r]["x"] - xo, np.inf) <= 1e-8 * np.linalg.norm(xo, np.inf)


def test_block_cyclic_lu_device_kernels():
    from oracle import densolve_oracle as O
    res = run_case("lu")
    n = 300
    A = np.asfortranarray(np.random.default_rng([0, n, 1]).uniform(-1.0, 1.0, (n, n)))
    W, piv, _ = O.lu_factor_blocked(A, 16)
    for r in (0, 1):
        assert np.array_equal(res[r]["piv"], piv)
        assert np.max(np.abs(res[r]["packed"] - W)) <= 1e-10 * np.max(np.abs(W))
