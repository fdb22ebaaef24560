"""Row-sharded CG (ds_cg_sharded) vs the fused single-GPU CG on the C4 matrix:
python tools/shard_rate.py [n] [iters] — devices=[0] (one shard: the sharded code path
with no peers) and devices=[0, 0] (two shards sharing GPU 0, exchanges live)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray, _padded_ld  # noqa: E402
from paper_1511_07207_b200.harness import generate_problem_device  # noqa: E402
from paper_1511_07207_b200.sharded import ShardedMatrix, ShardedVector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = SolverConfig(tolerance=1e-300, max_iterations=iters)
be = get_backend("b200")
dA, db, _ = generate_problem_device("spd", n, 0, "f64", be)
dx0 = DeviceArray(be.ctx, (n,), np.float64)
torch.as_tensor(dx0, device="cuda").zero_()
be.ctx.synchronize()


def rate(fn, reps=3):
    fn()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)  # each solve ends with a host sync
    return iters / best


x1, r1 = cg_solve(dA, db, dx0, cfg, be)
print(f"fused single-GPU CG      : {rate(lambda: cg_solve(dA, db, dx0, cfg, be)):8.1f} it/s")
tA, tb = torch.as_tensor(dA, device="cuda"), torch.as_tensor(db, device="cuda")
for devs in ([0], [0, 0]):
    sb = get_backend("b200", devices=devs)
    ss = sb.shardset(n, np.float64)
    blocks, bs, xs = [], [], []
    for ctx, q in zip(ss.ctxs, ss.ranks):
        r0, r1_ = ss.rows(q)
        blk = DeviceArray(ctx, (ss.n_loc, n), np.float64, ld=_padded_ld(ss.n_loc))
        bp = DeviceArray(ctx, (ss.n_loc,), np.float64)
        xp = DeviceArray(ctx, (ss.n_loc,), np.float64)
        t = torch.as_tensor(blk, device="cuda")
        t.zero_()
        t[: r1_ - r0].copy_(tA[r0:r1_, :])
        tbp = torch.as_tensor(bp, device="cuda")
        tbp.zero_()
        tbp[: r1_ - r0].copy_(tb[r0:r1_])
        torch.as_tensor(xp, device="cuda").zero_()
        blocks.append(blk), bs.append(bp), xs.append(xp)
    torch.cuda.synchronize()
    A_sh, b_sh, x0_sh = ShardedMatrix(ss, blocks), ShardedVector(ss, bs), ShardedVector(ss, xs)
    xd, rep = cg_solve(A_sh, b_sh, x0_sh, cfg, sb)
    xh = xd.to_host()
    print(f"sharded devices={devs!s:8}: {rate(lambda: cg_solve(A_sh, b_sh, x0_sh, cfg, sb)):8.1f} it/s  "
          f"history == fused[:4]? {np.allclose(rep.residual_history[:4], r1.residual_history[:4], rtol=1e-10)}  "
          f"|x - x_fused|/|x| = {np.linalg.norm(xh - x1.to_host()) / np.linalg.norm(x1.to_host()):.2e}")
    del A_sh, blocks
    sb.close()
    torch.cuda.empty_cache()
