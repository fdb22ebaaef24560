"""LU step timeline: python tools/lu_timeline.py [n] -- prints the library's
DENSOLVE_LU_TIMELINE report (main-stream interval per outer panel, side-stream look-ahead
factorization per outer panel) for one factorization after a warm-up, plus the wall time."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1511_07207_b200 import get_backend, lu_factor_blocked  # noqa: E402
from paper_1511_07207_b200.harness import generate_problem_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
be = get_backend("b200")
dA, _, _ = generate_problem_device("uniform", n, 1, "f64", be, rhs=False)
lu_factor_blocked(dA, 64, be)
for rep in range(2):
    be.ctx.synchronize()
    t0 = time.perf_counter()
    lu_factor_blocked(dA, 64, be)
    be.ctx.synchronize()
    print(f"n={n} wall {1e3 * (time.perf_counter() - t0):.2f} ms  "
          f"{2 * n ** 3 / 3 / (time.perf_counter() - t0) / 1e12:.2f} TFLOP/s", flush=True)
os.environ["DENSOLVE_LU_TIMELINE"] = "1"
lu_factor_blocked(dA, 64, be)
be.ctx.synchronize()
