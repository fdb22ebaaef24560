"""Per-phase timestamps of single LU panels (DENSOLVE_PANEL_TRACE=kb):
python tools/panel_trace.py n kb1 kb2 ...   (prints '[panel trace]' lines on stderr)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import get_backend, lu_factor_blocked  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402

be = get_backend("b200")
ctx = be.ctx
n = int(sys.argv[1])
g = torch.Generator(device="cuda")
g.manual_seed(1)
At = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2.0).sub_(1.0)
dA = DeviceArray(ctx, (n, n), np.float64)
for la in ("0", "1"):
    os.environ["DENSOLVE_LU_LOOKAHEAD"] = la
    for kb in sys.argv[2:]:
        os.environ["DENSOLVE_PANEL_TRACE"] = kb
        ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 8 * n * n)
        print(f"lookahead={la} kb={kb}", file=sys.stderr, flush=True)
        lu_factor_blocked(dA, 64, be)
        ctx.synchronize()
