import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1511_07207_b200 import lu_factor_blocked, lu_factor_unblocked, get_backend
be = get_backend("b200")
rng = np.random.default_rng(1234)
A = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(24, 24)))
ref = lu_factor_unblocked(A, be)
blk = lu_factor_blocked(A, 24, be)
d = np.argwhere(ref.packed != blk.packed)
print("mismatches", len(d), d[:10].tolist())
print("ref ptr", hex(ref.device.ptr), "blk ptr", hex(blk.device.ptr))
for n in (24, 100, 300):
    A = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(n, n)))
    f1 = lu_factor_blocked(A, 64, be); f2 = lu_factor_blocked(A, 64, be)
    print(n, "repeat equal", np.array_equal(f1.packed, f2.packed), np.array_equal(f1.pivots, f2.pivots))
