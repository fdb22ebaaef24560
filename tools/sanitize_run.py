"""Small runs of every solver for compute-sanitizer (memcheck / racecheck / synccheck): compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1511_07207_b200 import SolverConfig, get_backend, gmres_solve, cg_solve, lu_factor_blocked, lu_solve, bicgstab_solve, cholesky_factor
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem
be = get_backend("b200")
for n, m in ((200, 30), (64, 5)):
    A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=3, precision="f64"))
    x, r = gmres_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10, restart_m=m), be)
    print("gmres", n, m, r.iterations, r.converged, flush=True)
A, b, _ = generate_problem(ProblemSpec(kind="spd", n=300, seed=1, precision="f64"))
x, r = cg_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10), be); print("cg", r.iterations, flush=True)
x, r = bicgstab_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10), be); print("bicgstab", r.iterations, flush=True)
A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=700, seed=2, precision="f64"))
f = lu_factor_blocked(A, 64, be); x = lu_solve(f, b); print("lu", np.linalg.norm(A @ x - b), flush=True)
A, b, _ = generate_problem(ProblemSpec(kind="spd", n=600, seed=2, precision="f64"))
f = cholesky_factor(A, 64, be); print("chol ok", flush=True)
