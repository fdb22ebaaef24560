"""Row-sharded GMRES (ds_gmres_sharded) vs the fused single-GPU GMRES, one full cycle:
python tools/shard_gmres_rate.py [n] [m] [f32|f64]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import SolverConfig, get_backend, gmres_solve  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray, _padded_ld  # noqa: E402
from paper_1511_07207_b200.harness import generate_problem_device  # noqa: E402
from paper_1511_07207_b200.sharded import ShardedMatrix, ShardedVector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
m = int(sys.argv[2]) if len(sys.argv) > 2 else 50
prec = sys.argv[3] if len(sys.argv) > 3 else "f32"
dt = np.float32 if prec == "f32" else np.float64
cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
be = get_backend("b200")
dA, db, _ = generate_problem_device("general_nonsymmetric", n, 0, prec, be)
dx0 = DeviceArray(be.ctx, (n,), dt)
torch.as_tensor(dx0, device="cuda").zero_()
be.ctx.synchronize()


def rate(fn, reps=3):
    fn()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return m / best


x1, r1 = gmres_solve(dA, db, dx0, cfg, be)
print(f"fused single-GPU GMRES({m}) n={n} {prec}: {rate(lambda: gmres_solve(dA, db, dx0, cfg, be)):8.1f} it/s")
tA, tb = torch.as_tensor(dA, device="cuda"), torch.as_tensor(db, device="cuda")
for devs in ([0], [0, 0]):
    sb = get_backend("b200", devices=devs)
    ss = sb.shardset(n, dt)
    blocks, bs, xs = [], [], []
    for ctx, q in zip(ss.ctxs, ss.ranks):
        r0, r1_ = ss.rows(q)
        blk = DeviceArray(ctx, (ss.n_loc, n), dt, ld=_padded_ld(ss.n_loc))
        bp = DeviceArray(ctx, (ss.n_loc,), dt)
        xp = DeviceArray(ctx, (ss.n_loc,), dt)
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
    xd, rep = gmres_solve(A_sh, b_sh, x0_sh, cfg, sb)
    xh = xd.to_host()
    x1h = x1.to_host()
    print(f"sharded devices={devs!s:8}: {rate(lambda: gmres_solve(A_sh, b_sh, x0_sh, cfg, sb)):8.1f} it/s  "
          f"est[:3] rel diff {np.max(np.abs(np.array(rep.residual_history[:3]) - np.array(r1.residual_history[:3])) / np.array(r1.residual_history[:3])):.1e}  "
          f"|x - x_fused|/|x| = {np.linalg.norm(xh - x1h) / np.linalg.norm(x1h):.2e}")
    del A_sh, blocks
    sb.close()
    torch.cuda.empty_cache()
