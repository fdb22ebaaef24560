"""Two DMMA GEMMs running at the same time on two streams (two library contexts) vs the
same GEMMs run one after the other: python tools/gemm_concurrent.py"""
import os
import sys
from ctypes import c_void_p

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import _lib  # noqa: E402

c1, c2 = _lib.Context(0), _lib.Context(0)
OTHER = os.environ.get("OTHER", "gemm")  # what runs on the second stream: gemm | gemv
n, K = 8192, 512
g = torch.Generator(device="cuda").manual_seed(3)
mats = []
for _ in range(2):
    A = torch.rand((K, n), dtype=torch.float64, device="cuda", generator=g)  # column-major n x K (ld n)
    B = torch.rand((n, K), dtype=torch.float64, device="cuda", generator=g)  # column-major K x n (ld K)
    C = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    mats.append((A, B, C))
torch.cuda.synchronize()


def run(ctx, A, B, C, out):
    _lib.check(ctx.lib.ds_gemm(ctx.handle, _lib.DS_F64, n, n, K, -1.0, c_void_p(A.data_ptr()), n, c_void_p(B.data_ptr()),
                               K, 1.0, c_void_p(C.data_ptr()), n, c_void_p(out.data_ptr()), n))


ref = [torch.empty_like(m[2]) for m in mats]
gv = torch.empty(n, dtype=torch.float64, device="cuda")
run(c1, *mats[0], ref[0]); c1.synchronize()
run(c1, *mats[1], ref[1]); c1.synchronize()
bad = 0
for trial in range(int(os.environ.get("TRIALS", "20"))):
    outs = [torch.empty_like(m[2]) for m in mats]
    run(c1, *mats[0], outs[0])
    if OTHER == "gemm":
        run(c2, *mats[1], outs[1])
    else:
        outs[1] = ref[1]
        for _ in range(8):
            A1 = mats[1][2]
            _lib.check(c2.lib.ds_gemv(c2.handle, _lib.DS_F64, n, n, c_void_p(A1.data_ptr()), n,
                                      c_void_p(mats[1][0].data_ptr()), c_void_p(outs[0].data_ptr() if False else gv.data_ptr())))
    c1.synchronize(); c2.synchronize()
    for i in range(2):
        if not torch.equal(outs[i], ref[i]):
            bad += 1
            print(f"trial {trial} gemm {i}: max diff {(outs[i] - ref[i]).abs().max().item():.3e}")
print("concurrent GEMMs bitwise equal to sequential" if bad == 0 else f"{bad} mismatches")
