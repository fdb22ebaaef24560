"""GMRES per-call cost split: one-cycle calls at m = 5, 10, 30, 60 for n = 4096 and 256, so
t = fixed + m * per_step separates the call overhead from the Arnoldi step.
python tools/gmres_overhead.py"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1511_07207_b200 import SolverConfig, get_backend, gmres_solve
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem
be = get_backend("b200"); ctx = be.ctx
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
for n in (4096, 256):
    A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=0, precision="f64"))
    dA, db, dx0 = be.stage_in(A, b, np.zeros_like(b))
    for m in (5, 10, 30, 60):
        cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
        gmres_solve(dA, db, dx0, cfg, be); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record(stream)
        for _ in range(20):
            x, rep = gmres_solve(dA, db, dx0, cfg, be)
        e1.record(stream); torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"n={n} m={m}: {e0.elapsed_time(e1)/20:.3f} ms/call (events), host {1e3*(t1-t0)/20:.3f} ms/call", flush=True)
