"""LU factors with the TMA-fed vs the cp.async GEMM (separate processes; the switch is read
once): python tools/lu_tma_check.py run out.npz n  |  python tools/lu_tma_check.py cmp a.npz b.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for key in a.files:
        x, y = a[key], b[key]
        if x.shape != y.shape:
            print(key, "shape differs")
            continue
        d = np.abs(x.astype(np.float64) - y.astype(np.float64))
        bad = np.argwhere(d > 0)
        print(key, "bitwise equal" if len(bad) == 0 else f"{len(bad)} differ, max {d.max():.3e}, first {bad[:3].tolist()}")
    sys.exit(0)
from paper_1511_07207_b200 import get_backend, lu_factor_blocked  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402

n = int(sys.argv[3])
be = get_backend("b200")
A = np.asfortranarray(np.random.default_rng(n).uniform(-1, 1, (n, n)))
out = {}
for la in ("1", "0"):
    os.environ["DENSOLVE_LU_LOOKAHEAD"] = la
    f = lu_factor_blocked(A, 64, be)
    out[f"piv_la{la}"] = np.asarray(f.pivots)
    out[f"lu_la{la}"] = f.packed
np.savez(sys.argv[2], **out)
print("saved", sys.argv[2])
