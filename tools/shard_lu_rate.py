"""Block-cyclic LU (ds_lu_block_cyclic) vs the single-GPU LU: python tools/shard_lu_rate.py n"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import get_backend, lu_factor_blocked  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = np.asfortranarray(np.random.default_rng(1).uniform(-1, 1, (n, n)))
for devs in (None, [0, 0]):
    be = get_backend("b200") if devs is None else get_backend("b200", devices=devs)
    f0 = lu_factor_blocked(A, 64, be)
    best = 1e30
    for _ in range(2):
        t0 = time.perf_counter()
        f = lu_factor_blocked(A, 64, be)
        best = min(best, time.perf_counter() - t0)
    same = np.array_equal(np.asarray(f.pivots), np.asarray(f0.pivots))
    print(f"LU n={n} {'single GPU' if devs is None else 'devices=' + str(devs)}: {best * 1e3:.1f} ms incl. host "
          f"transfers ({2 / 3 * n ** 3 / best / 1e12:.2f} TFLOP/s), repeatable pivots {same}", flush=True)
