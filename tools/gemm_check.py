"""Bitwise equality of GEMM kernel variants on ragged shapes:
DENSOLVE_GEMM_TMA=0 python tools/gemm_check.py out0.npz; python tools/gemm_check.py out1.npz;
python tools/gemm_check.py --compare out0.npz out1.npz.  A third argument f32 checks the fp32
path (DENSOLVE_GEMM32_SMALL=1 selects the 64 x 64 kernel)."""
import os
import sys
from ctypes import c_void_p

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [(128, 64, 16), (300, 200, 37), (1000, 513, 512), (4096, 4096, 512), (257, 1031, 64), (64, 64, 1),
          (130, 66, 18), (2048, 448, 64)]

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise equal" if not bad else f"DIFFER: {bad}")
    sys.exit(1 if bad else 0)

from paper_1511_07207_b200 import _lib, get_backend  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402

dt = np.float32 if len(sys.argv) > 2 and sys.argv[2] == "f32" else np.float64
code = _lib.DS_F32 if dt == np.float32 else _lib.DS_F64
tol = 1e-4 if dt == np.float32 else 1e-13
be = get_backend("b200")
ctx = be.ctx
rng = np.random.default_rng(5)
out = {}
for (m, n, k) in SHAPES:
    for mode, (alpha, beta) in (("sub", (-1.0, 1.0)), ("gen", (0.75, -1.25))):
        A = np.asfortranarray(rng.standard_normal((m, k)).astype(dt))
        B = np.asfortranarray(rng.standard_normal((k, n)).astype(dt))
        C = np.asfortranarray(rng.standard_normal((m, n)).astype(dt))
        dA, dB, dC = DeviceArray.from_host(A, ctx), DeviceArray.from_host(B, ctx), DeviceArray.from_host(C, ctx)
        dO = DeviceArray(ctx, (m, n), dt)
        _lib.check(ctx.lib.ds_gemm(ctx.handle, code, m, n, k, alpha, c_void_p(dA.ptr), dA.ld, c_void_p(dB.ptr),
                                   dB.ld, beta, c_void_p(dC.ptr), dC.ld, c_void_p(dO.ptr), dO.ld))
        o = dO.to_host()
        ref = beta * C.astype(np.float64) + alpha * (A.astype(np.float64) @ B.astype(np.float64))
        err = np.abs(o - ref).max() / max(1.0, np.abs(ref).max()) / max(1.0, np.sqrt(k))
        assert err < tol, (m, n, k, mode, err)
        out[f"{m}x{n}x{k}_{mode}"] = o
np.savez(sys.argv[1], **out)
print("saved", len(out), "results; all within", tol, "(x sqrt k) of numpy fp64")
