"""Pinned host->device copy rate with and without binding the process to the GPU's NVML CPU
affinity (first-touch places the pinned pages on the allocating thread's NUMA node):
python tools/h2d_affinity.py"""
import os
import time

import torch

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
local = [w * 64 + b for w, m in enumerate(words) for b in range(64) if m >> b & 1]
print("cpus", os.cpu_count(), "gpu-local", len(local), local[:8], "...", "current", len(os.sched_getaffinity(0)))
nb = 2 << 30


def rate(tag):
    src = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    src.fill_(1)
    dst = torch.empty(nb, dtype=torch.uint8, device="cuda")
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(4):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    print(tag, f"{4 * nb / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)


rate("default affinity")
os.sched_setaffinity(0, local)
rate("gpu-local affinity")
other = sorted(set(range(os.cpu_count())) - set(local))
if other:
    os.sched_setaffinity(0, other)
    rate("remote affinity")
