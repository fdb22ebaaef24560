import os, sys, time
sys.path.insert(0, "/root/repo")
os.environ.setdefault("RANK","0"); os.environ.setdefault("WORLD_SIZE","1"); os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29561")
import torch, numpy as np
import torch.distributed as dist
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=dev)
from paper_1511_07207_b200 import SolverConfig
from paper_1511_07207_b200.distributed import CudaShardOps, TorchComm, cg_solve_sharded, spd_block_device
n = 8192
ops = CudaShardOps(); comm = TorchComm()
stream = torch.cuda.current_stream()
ops.bind_current_stream()
A_blk = spd_block_device(n, 0, n, torch, dev)
b = torch.rand(n, dtype=torch.float64, device=dev); x0 = torch.zeros_like(b)
cfg = SolverConfig(tolerance=1e-300, max_iterations=200)
cg_solve_sharded(A_blk, b, x0, n, cfg, comm, ops)
torch.cuda.synchronize()
for its in (100, 200):
    cfg = SolverConfig(tolerance=1e-300, max_iterations=its)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    cg_solve_sharded(A_blk, b, x0, n, cfg, comm, ops, check_sym=False)
    e1.record(); torch.cuda.synchronize()
    print(its, "its:", e0.elapsed_time(e1), "ms gpu,", (time.perf_counter()-t0)*1e3, "ms wall", flush=True)
from torch.profiler import profile, ProfilerActivity
cfg = SolverConfig(tolerance=1e-300, max_iterations=50)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    cg_solve_sharded(A_blk, b, x0, n, cfg, comm, ops, check_sym=False)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14))
dist.destroy_process_group()
