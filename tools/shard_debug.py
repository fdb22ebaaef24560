"""Run one sharded-CG configuration (devices list, n) in this process and report the time:
python tools/shard_debug.py 0,0,0,0 257"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import densolve_oracle as O  # noqa: E402
from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend  # noqa: E402

devs = [int(d) for d in sys.argv[1].split(",")]
n = int(sys.argv[2])
A, b, _ = O.generate_problem("spd", n, 7)
be = get_backend("b200", devices=devs)
for rep_i in range(2):
    t0 = time.perf_counter()
    try:
        x, rep = cg_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10), be)
        xo, ro = O.cg(A, b, np.zeros_like(b), 1e-10)
        print(f"devices={devs} n={n}: {time.perf_counter() - t0:.3f} s, it {rep.iterations} vs {ro['iterations']}, "
              f"err {np.linalg.norm(x - xo, np.inf) / np.linalg.norm(xo, np.inf):.2e}", flush=True)
    except Exception as e:
        print(f"devices={devs} n={n}: FAILED after {time.perf_counter() - t0:.3f} s: {e}", flush=True)
        break
