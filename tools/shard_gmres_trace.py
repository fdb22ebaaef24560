"""Host-side timeline of one sharded GMRES cycle (DENSOLVE_SHARD_TRACE) + device time:
python tools/shard_gmres_trace.py n m prec"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import SolverConfig, get_backend, gmres_solve  # noqa: E402
from paper_1511_07207_b200.harness import generate_problem_device  # noqa: E402

n, m, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
dt = np.float32 if prec == "f32" else np.float64
be = get_backend("b200")
dA, db, _ = generate_problem_device("general_nonsymmetric", n, 0, prec, be)
A, b = dA.to_host(), db.to_host()
del dA
sb = get_backend("b200", devices=[0])
sA, sbv, sx0 = sb.stage_in(A, b, np.zeros_like(b))
del A
cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
gmres_solve(sA, sbv, sx0, cfg, sb)
for trial in range(2):
    t0 = time.perf_counter()
    x, rep = gmres_solve(sA, sbv, sx0, cfg, sb)
    print(f"trial {trial}: {time.perf_counter() - t0:.4f} s, {rep.iterations} its, launches {rep.kernel_launches}",
          flush=True)
