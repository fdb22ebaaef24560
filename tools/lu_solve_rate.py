"""lu_solve / substitution timing at n (default 16384): python tools/lu_solve_rate.py [n] [f64|f32]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1511_07207_b200 import (backward_substitution, forward_substitution, get_backend,  # noqa: E402
                                   lu_factor_blocked, lu_solve)
from paper_1511_07207_b200.harness import generate_problem_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
be = get_backend("b200")
dA, db, dx = generate_problem_device("uniform", n, 1, prec, be)
f = lu_factor_blocked(dA, 64, be)


def rate(fn, reps=10):
    fn()
    be.ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    be.ctx.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out
# (host wall time around `reps` back-to-back calls, each with its own host synchronisation)


ms, x = rate(lambda: lu_solve(f, db))
err = float(np.max(np.abs(x.to_host() - dx.to_host())))
import hashlib  # noqa: E402
h = hashlib.sha256(np.ascontiguousarray(x.to_host()).tobytes()).hexdigest()[:16]
print(f"{prec} n={n} lu_solve {ms:.3f} ms  {8.0 * n * n / ms / 1e6:.1f} GB/s  err {err:.2e}  x sha256 {h}")
ms, _ = rate(lambda: forward_substitution(f.device, db, unit_diagonal=True))
print(f"forward (unit) {ms:.3f} ms  {4.0 * n * n / ms / 1e6:.1f} GB/s")
ms, _ = rate(lambda: backward_substitution(f.device, db))
print(f"backward {ms:.3f} ms  {4.0 * n * n / ms / 1e6:.1f} GB/s")
