#!/usr/bin/env python
"""Benchmark of the B200 densolve hot path (BASELINE.json metric).

Headline (``value``): CG iterations/s on a dense SPD n=32768 fp64 system
(config C4) with A resident in HBM; one *step* = one ``cg_solve`` call with
tolerance 1e-300 and max_iterations=ITERS (the reference's own fixed-iteration
idiom, tests/test_krylov.py:188-191), i.e. symmetry gate + setup + ITERS
iterations.  ``e2e`` is the same metric through the public API with pinned
HOST buffers (A, b, x0 uploaded and x downloaded inside every step).
``components`` adds GMRES(30) n=4096 fp64 (C2) and GMRES(50) n=65536 fp32 (C5),
one full cycle per step; blocked LU (b=64) fp64 GFLOP/s at n=16384 (C3) and
n=32768 (C5 per-GPU size); BiCGSTAB and Cholesky on the C4 matrix.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--impl reference times the reference CPU path (the NumPy restatement in
oracle/, which makes the same NumPy/BLAS calls as the reference package) on
the host cores, same metric and workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "CG/GMRES iters/sec & HBM GB/s; LU GFLOP/s at n=32768, 1/2/4/8 B200 vs CPU"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6551.0)), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


FP64_PEAK_TFLOPS = 37.1  # DMMA/DFMA measured on this pool (profiles/fp64_peak_r01.txt)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML every 20 ms
    from a thread (nvidia-smi -lms as the fallback, whose ~1 s start-up leaves few
    samples in a sub-second region)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int = 0, period_s: float = 0.02):
        self.index = index
        self.period = period_s
        self.rows = []  # (sm_mhz, sm_max_mhz, set(reasons))
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def sample():
                sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, smax, {nm for nm, bit in zip(self.NAMES, bits) if rs & bit}))

            sample()  # fail here, not in the thread, if NVML cannot read this device
            self.nvml = pynvml

            def loop():
                while not self.stop.wait(self.period):
                    try:
                        sample()
                    except Exception:  # noqa: BLE001 - sampling is best effort
                        return
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            self.rows = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((float(r[0]), float(r[1]),
                                  {nm for nm, v in zip(self.NAMES, r[3:7]) if v.lower().startswith("active")}))
            except (ValueError, IndexError):
                continue

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
            try:
                self.nvml.nvmlShutdown()
            except Exception:  # noqa: BLE001
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = set().union(*[r[2] for r in self.rows])
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.rows[-1][1], "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------- helpers
def lib_matvec(be, A_t, x_t):
    """y = colmajor(A_t) @ x with the library's own GEMV (no cuBLAS even in the setup);
    torch's row-major A_t read as column-major is A_t^T."""
    from ctypes import c_void_p
    import torch
    from paper_1511_07207_b200 import _lib
    n = x_t.shape[0]
    code = _lib.DS_F64 if x_t.dtype == torch.float64 else _lib.DS_F32
    y = torch.empty_like(x_t)
    torch.cuda.synchronize()
    _lib.check(be.ctx.lib.ds_gemv(be.ctx.handle, code, n, n, c_void_p(A_t.data_ptr()), n,
                                  c_void_p(x_t.data_ptr()), c_void_p(y.data_ptr())))
    be.ctx.synchronize()
    return y


def spd_fast_device(n, seed, torch, device, be):
    """Synthetic dense SPD: A = (R + R^T)/2 + sqrt(n) I, R ~ U[-1,1] (seeded, on the GPU).
    The symmetric part has a semicircle spectrum of radius ~0.82 sqrt(n), so
    lambda(A) in ~[0.18, 1.82] sqrt(n): SPD with kappa ~ 10, which keeps a
    fixed 100-iteration CG far from underflow (rate ~0.5 per iteration)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    A = torch.rand((n, n), dtype=torch.float64, device=device, generator=g)
    A.mul_(2.0).sub_(1.0)
    A.add_(A.t().clone()).mul_(0.5)
    A.diagonal().add_(float(n) ** 0.5)
    xt = torch.rand(n, dtype=torch.float64, device=device, generator=g).mul_(2.0).sub_(1.0)
    return A, lib_matvec(be, A, xt)  # A symmetric: row-major == column-major


def spd_fast_host(n, seed):
    rng = np.random.default_rng([seed, n, 2])
    A = rng.uniform(-1.0, 1.0, size=(n, n))
    A += A.T.copy()
    A *= 0.5
    A[np.diag_indices(n)] += float(n) ** 0.5
    xt = rng.uniform(-1.0, 1.0, size=n)
    return np.asfortranarray(A), A @ xt


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import densolve_oracle as O

    n = args.n
    # bounded sample: ~0.35 s per CPU iteration at n=32768, keep the whole run near 3 minutes
    iters = max(10, min(args.iters, int(180.0 / ((args.steps + 1) * 0.35))))
    cores = os.cpu_count() or 1
    A, b = spd_fast_host(n, 0)
    x0 = np.zeros(n)
    times = []
    for k in range(min(args.warmup, 1) + args.steps):
        t0 = time.perf_counter()
        O.cg(A, b, x0, 1e-300, iters, O.Ops(threads=cores))
        dt = time.perf_counter() - t0
        if k >= min(args.warmup, 1):
            times.append(dt)
    tot = sum(times)
    val = iters * len(times) / tot
    line = {"impl": "reference", "metric": BASELINE_METRIC, "value": val,
            "unit": f"CG iters/s (n={n} fp64)", "n_gpus": ws, "steps": args.steps,
            "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C4 CG dense SPD n={n} fp64, fixed iterations per step (bounded CPU sample)",
                       "n": n, "iters_per_step": iters, "b200_arm_iters_per_step": args.iters},
            "cpu_baseline": {"value": val, "unit": f"CG iters/s (n={n} fp64)", "cores": cores, "kind": "port",
                             "sample": f"oracle.cg (NumPy/OpenBLAS restatement of krylov.cg_solve incl. "
                                       f"symmetry gate), n={n}, {iters} iterations per step"},
            "e2e": {"value": val, "unit": f"CG iters/s (n={n} fp64)", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- B200 arm
def cpu_baseline_sample(n, iters):
    from oracle import densolve_oracle as O

    cores = os.cpu_count() or 1
    A, b = spd_fast_host(n, 0)
    t0 = time.perf_counter()
    O.cg(A, b, np.zeros(n), 1e-300, iters, O.Ops(threads=cores))
    dt = time.perf_counter() - t0
    del A
    return {"value": iters / dt, "unit": f"CG iters/s (n={n} fp64)", "cores": cores, "kind": "port",
            "sample": f"one step: oracle.cg (NumPy/OpenBLAS restatement of krylov.cg_solve incl. symmetry "
                      f"gate) at n={n}, {iters} iterations, {dt:.1f} s"}


def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = ws > 1 or args.force_sharded
    if sharded:
        import torch.distributed as dist
        if not dist.is_initialized():
            # --force-sharded without torchrun: a world of one on 127.0.0.1
            for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"),
                         ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531")):
                os.environ.setdefault(k, v)
            dist.init_process_group("nccl", device_id=dev)
    from paper_1511_07207_b200 import (SolverConfig, cg_solve, get_backend, gmres_solve,
                                       lu_factor_blocked, pinned_empty)
    from paper_1511_07207_b200.device import DeviceArray
    from paper_1511_07207_b200.harness import ProblemSpec, generate_problem

    be = get_backend("b200", device=local)
    ctx = be.ctx
    stream = torch.cuda.Stream(dev)  # a real (non-legacy) stream shared with the library
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)  # all library work on this stream: the events see it
    hbm_peak, peak_src = _peaks()
    n, iters = args.n, args.iters
    cfg = SolverConfig(tolerance=1e-300, max_iterations=iters)

    if sharded:
        try:
            return bench_sharded_cg(args, torch, dev, be)
        finally:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()

    # ---- inputs: synthetic SPD generated on the device, staged into a DeviceArray
    At, bt = spd_fast_device(n, 0, torch, dev, be)
    dA = DeviceArray(ctx, (n, n), np.float64)
    assert dA.ld == n
    ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 8 * n * n)
    db = DeviceArray(ctx, (n,), np.float64)
    ctx.lib.ds_memcpy_d2d(ctx.handle, db.ptr, bt.data_ptr(), 8 * n)
    dx0 = DeviceArray(ctx, (n,), np.float64)
    ctx.lib.ds_memset(ctx.handle, dx0.ptr, 0, 8 * n)
    # host copies (pinned) for the end-to-end arm
    A_h = pinned_empty((n, n), np.float64, order="F")
    A_h_t = torch.from_numpy(A_h.reshape(-1, order="F").view(np.float64))
    A_h_t.copy_(At.reshape(-1))  # A is symmetric: row-major bytes == column-major bytes
    b_h = pinned_empty((n,), np.float64)
    b_h[:] = bt.cpu().numpy()
    x0_h = pinned_empty((n,), np.float64)
    x0_h[:] = 0.0
    del At
    torch.cuda.synchronize()

    # ---- headline: device-resident fixed-iteration CG steps
    for _ in range(args.warmup):
        cg_solve(dA, db, dx0, cfg, be)
    torch.cuda.synchronize()
    def timed_region():
        l0 = ctx.launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                x, rep = cg_solve(dA, db, dx0, cfg, be)
            e1.record(stream)
            torch.cuda.synchronize()
        return x, rep, ctx.launches() - l0, e0.elapsed_time(e1), clk

    x, rep, launches, ms, clk = timed_region()
    remeasured = False
    if set(clk.summary()["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}:
        # a throttled region is rejected and measured once more (sw_power_cap is kept, noted)
        x, rep, launches, ms, clk = timed_region()
        remeasured = True
    assert rep.iterations == iters
    value = iters * args.steps / (ms / 1e3)

    # ---- roofline of the dominant kernel (GEMV stream of A): timed alone, same stream
    from ctypes import c_void_p
    from paper_1511_07207_b200 import _lib
    dy = DeviceArray(ctx, (n,), np.float64)
    R = 20

    def gemv():
        _lib.check(ctx.lib.ds_gemv(ctx.handle, _lib.DS_F64, n, n, c_void_p(dA.ptr), dA.ld,
                                   c_void_p(db.ptr), c_void_p(dy.ptr)))

    for _ in range(3):
        gemv()
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(R):
        gemv()
    g1.record(stream)
    torch.cuda.synchronize()
    gemv_ms = g0.elapsed_time(g1) / R
    gemv_bytes = 8.0 * (n * n + 2 * n)
    achieved = gemv_bytes / (gemv_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_gemv_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "kernel": "gemv_partial_kernel<double,2,8> + gemv_reduce (ds_gemv)",
                "algorithmic_bytes_per_launch": gemv_bytes, "avg_launch_ms": round(gemv_ms, 4),
                "peak_source": peak_src,
                "cg_iteration_GBps": round(8.0 * (n * n + 10 * n) / (ms / 1e3 / (iters * args.steps)) / 1e9, 1)}

    # ---- end to end through the public API with pinned host buffers.  Every step copies
    # A, b, x0 host->device and x (plus the history) back.  Pipelined (the value): the next
    # step's operands are staged with B200Backend.stage_in_async into the other of two
    # device buffer sets while this step solves (copy stream || compute stream).  The
    # serial variant (upload, solve, download in turn) is reported beside it.
    for _ in range(max(1, min(args.warmup, 2))):
        cg_solve(A_h, b_h, x0_h, cfg, be)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        x_h, rep_h = cg_solve(A_h, b_h, x0_h, cfg, be)
    f1.record(stream)
    torch.cuda.synchronize()
    serial_ms = max(f0.elapsed_time(f1), 1e3 * (time.perf_counter() - t0))
    del dx0  # free the resident operands' x0; A stays for the components below
    bufs = [(DeviceArray(ctx, (n, n), np.float64), DeviceArray(ctx, (n,), np.float64),
             DeviceArray(ctx, (n,), np.float64)) for _ in range(2)]
    be.stage_in_async(A_h, b_h, x0_h, out=bufs[0])
    cg_solve(*bufs[0], cfg, be)  # warm-up of the pipelined path
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f0.record(stream)
    be.stage_in_async(A_h, b_h, x0_h, out=bufs[0])
    for s_ in range(args.steps):
        if s_ + 1 < args.steps:
            be.stage_in_async(A_h, b_h, x0_h, out=bufs[(s_ + 1) % 2])
        xd, rep_h = cg_solve(*bufs[s_ % 2], cfg, be)
        x_h = xd.to_host()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max(f0.elapsed_time(f1), 1e3 * (time.perf_counter() - t0))
    assert rep_h.iterations == iters
    e2e = {"value": iters * args.steps / (e2e_ms / 1e3), "unit": f"CG iters/s (n={n} fp64)",
           "h2d_bytes_per_step": int(A_h.nbytes + b_h.nbytes + x0_h.nbytes),
           "d2h_bytes_per_step": int(x_h.nbytes + 8 * (iters + 1)),
           "ms_per_step": e2e_ms / args.steps,
           "pipelining": "step s+1's H2D (stage_in_async, copy stream) overlaps step s's solve; 2 device buffer sets",
           "serial_value": iters * args.steps / (serial_ms / 1e3), "serial_ms_per_step": serial_ms / args.steps}
    del bufs
    dx0 = DeviceArray(ctx, (n,), np.float64)
    ctx.lib.ds_memset(ctx.handle, dx0.ptr, 0, 8 * n)
    del A_h, A_h_t

    components = {}
    if not args.only_cg:
        from paper_1511_07207_b200 import bicgstab_solve, cholesky_factor
        components["bicgstab"] = bench_bicgstab(args, torch, stream, be, dA, db, dx0, n, bicgstab_solve,
                                                SolverConfig, hbm_peak)
        components["cholesky"] = bench_cholesky(args, torch, stream, be, dA, n, cholesky_factor)
    del dA
    torch.cuda.empty_cache()
    if not args.only_cg:
        components["gmres_c2"] = bench_gmres(args, torch, stream, be, generate_problem, ProblemSpec,
                                             gmres_solve, SolverConfig)
        components["gmres_c5"] = bench_gmres_c5(args, torch, dev, stream, be, gmres_solve, SolverConfig,
                                                hbm_peak)
        components["lu_c3"] = bench_lu(args, torch, dev, stream, be, lu_factor_blocked, args.lu_n)
        components["lu_c5"] = bench_lu(args, torch, dev, stream, be, lu_factor_blocked, args.lu_n5)

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(n, min(iters, 30))  # ~15-25 s of host work

    line = {"metric": BASELINE_METRIC, "value": round(value, 3), "unit": f"CG iters/s (n={n} fp64)",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded dense SPD A=(R+R^T)/2+sqrt(n)I, R~U[-1,1], kappa~10, generated on device)",
            "config": {"workload": f"C4: CG dense SPD n={n} fp64, fixed {iters} iterations per step "
                                   f"(tolerance 1e-300), 1 GPU", "n": n, "iters_per_step": iters,
                       "l2_policy": f"inputs larger than L2 (A = {8 * n * n / 2**30:.1f} GiB >> 126 MB L2)",
                       "parallelism": f"rows{ws}"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": dict(clk.summary(), remeasured=remeasured), "components": components}
    print(json.dumps(line), flush=True)


def _timed(torch, stream, fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = None
    for _ in range(reps):
        out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def bench_gmres(args, torch, stream, be, generate_problem, ProblemSpec, gmres_solve, SolverConfig):
    """C2: GMRES(30) general_nonsymmetric n=4096 fp64 (the harness generator, host-built)."""
    n, m = 4096, 30
    A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=0))
    dA, db, dx0 = be.stage_in(A, b, np.zeros_like(b))
    cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
    ms, (x, rep) = _timed(torch, stream, lambda: gmres_solve(dA, db, dx0, cfg, be), 10)
    return {"workload": f"C2: GMRES({m}) general_nonsymmetric n={n} fp64, one full cycle per step "
                        "(residual + 30 Arnoldi steps + update + true residual)",
            "value": round(rep.iterations / (ms / 1e3), 1), "unit": "inner iters/s", "ms_per_step": round(ms, 4)}


def nonsym_fast_device(n, seed, torch, device, dtype, be):
    """Synthetic dense nonsymmetric A = R + 1.5 sqrt(n) I, R ~ U[-1,1] (seeded, on the GPU, in the
    target dtype; the harness recipe needs ~130 GB of fp64 temporaries at n=65536).  R's spectrum
    fills a disk of radius sqrt(n/3) (circular law), so GMRES contracts by ~0.38 per step: one
    full 50-step cycle stays far above the fp32 underflow of the Givens estimate."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    A = torch.empty((n, n), dtype=dtype, device=device)
    for c0 in range(0, n, 4096):  # column blocks keep the fp32 temporaries small
        blk = torch.rand((min(4096, n - c0), n), dtype=dtype, device=device, generator=g)
        A[c0:c0 + blk.shape[0]] = blk.mul_(2.0).sub_(1.0)
    A.diagonal().add_(1.5 * float(n) ** 0.5)
    xt = torch.rand(n, dtype=dtype, device=device, generator=g).mul_(2.0).sub_(1.0)
    return A, lib_matvec(be, A, xt)  # torch row-major A read column-major is A^T: b = A^T x


def bench_gmres_c5(args, torch, dev, stream, be, gmres_solve, SolverConfig, hbm_peak):
    """C5: GMRES(50) n=65536 fp32, one full cycle per step (HBM-capacity sizing, 1 GPU)."""
    from paper_1511_07207_b200.device import DeviceArray

    n, m = args.gmres_n, 50
    ctx = be.ctx
    At, bt = nonsym_fast_device(n, 3, torch, dev, torch.float32, be)
    dA = DeviceArray(ctx, (n, n), np.float32)
    ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 4 * n * n)
    db = DeviceArray(ctx, (n,), np.float32)
    ctx.lib.ds_memcpy_d2d(ctx.handle, db.ptr, bt.data_ptr(), 4 * n)
    dx0 = DeviceArray(ctx, (n,), np.float32)
    ctx.lib.ds_memset(ctx.handle, dx0.ptr, 0, 4 * n)
    del At, bt
    torch.cuda.synchronize()
    cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
    ms, (x, rep) = _timed(torch, stream, lambda: gmres_solve(dA, db, dx0, cfg, be), 3)
    # algorithmic bytes of one cycle: (m + 2) passes over A (m Arnoldi GEMVs + residual + true
    # residual) + per step k the basis traffic (2k + 7) n + the x update (m + 2) n
    s = 4.0
    byts = s * ((m + 2) * n * n + sum((2 * k + 7) * n for k in range(m)) + (m + 2) * n)
    gbs = byts / (ms / 1e3) / 1e9
    del dA
    torch.cuda.empty_cache()
    return {"workload": f"C5: GMRES({m}) dense nonsymmetric A = R + 1.5 sqrt(n) I, n={n} fp32 (device-generated), "
                        "one full cycle per step", "cycles": len(rep.restart_cycles or []), "value": round(rep.iterations / (ms / 1e3), 1),
            "unit": "inner iters/s", "ms_per_step": round(ms, 3), "GBps": round(gbs, 1),
            "frac_of_hbm_peak": round(gbs / hbm_peak, 4)}


def bench_bicgstab(args, torch, stream, be, dA, db, dx0, n, bicgstab_solve, SolverConfig, hbm_peak):
    """BiCGSTAB on the C4 matrix, fixed 50 iterations per step."""
    iters = 50
    cfg = SolverConfig(tolerance=1e-300, max_iterations=iters)
    ms, (x, rep) = _timed(torch, stream, lambda: bicgstab_solve(dA, db, dx0, cfg, be), 2)
    its = rep.iterations
    gbs = 8.0 * (2 * its + 1) * (n * n) / (ms / 1e3) / 1e9
    return {"workload": f"BiCGSTAB dense SPD n={n} fp64 (C4 matrix), fixed {iters} iterations per step",
            "value": round(its / (ms / 1e3), 2), "unit": "iters/s", "ms_per_step": round(ms, 3),
            "iterations": its, "breakdown": rep.breakdown, "GBps_A_stream": round(gbs, 1),
            "frac_of_hbm_peak": round(gbs / hbm_peak, 4)}


def bench_cholesky(args, torch, stream, be, dA, n, cholesky_factor):
    """Cholesky of the C4 SPD matrix, b=64, device-resident."""
    runs = [_timed(torch, stream, lambda: cholesky_factor(dA, 64, be), 1)[0] for _ in range(3)]
    ms = min(runs)  # 1 warm-up (inside _timed) + best of 3, harness.py:281-294
    tf = n ** 3 / 3.0 / (ms / 1e3) / 1e12
    return {"workload": f"blocked Cholesky b=64, dense SPD n={n} fp64 (C4 matrix), device-resident; best of 3",
            "value": round(tf * 1e3, 1), "unit": "GFLOP/s", "ms": round(ms, 2),
            "ms_runs": [round(r, 2) for r in runs],
            "fp64_peak_tflops": FP64_PEAK_TFLOPS, "frac_of_fp64_peak": round(tf / FP64_PEAK_TFLOPS, 4)}


def bench_lu(args, torch, dev, stream, be, lu_factor_blocked, n):
    from paper_1511_07207_b200.device import DeviceArray

    ctx = be.ctx
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    At = torch.rand((n, n), dtype=torch.float64, device=dev, generator=g).mul_(2.0).sub_(1.0)
    dA = DeviceArray(ctx, (n, n), np.float64)
    ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 8 * n * n)
    del At
    torch.cuda.synchronize()
    f = lu_factor_blocked(dA, 64, be)  # warm-up
    del f
    # 1 warm-up + best-of-3, the reference's own timing protocol (harness.py:281-294)
    runs = [_timed(torch, stream, lambda: lu_factor_blocked(dA, 64, be), 1)[0] for _ in range(3)]
    ms = min(runs)
    del dA
    torch.cuda.empty_cache()
    flops = 2.0 * n ** 3 / 3.0
    tf = flops / (ms / 1e3) / 1e12
    return {"workload": f"blocked LU b=64, uniform U[-1,1] n={n} fp64 (pivoting family), device-resident "
                        "(includes the device copy of A, direct.py:61); best of 3 after 1 warm-up",
            "value": round(tf * 1e3, 1), "unit": "GFLOP/s", "ms": round(ms, 2),
            "ms_runs": [round(r, 2) for r in runs],
            "fp64_peak_tflops": FP64_PEAK_TFLOPS, "frac_of_fp64_peak": round(tf / FP64_PEAK_TFLOPS, 4)}


# ---------------------------------------------------------------------------- N > 1 (torchrun)
def bench_sharded_cg(args, torch, dev, be):
    """`bench.py --gpus N` under torchrun: C4 CG row-sharded over N GPUs (strong scaling).
    Same JSON contract as the 1-GPU line: device-resident `value` (max over ranks of the
    CUDA-event time), `e2e` (each rank uploads its row block of A, b, x0 from pinned host
    memory and downloads its x shard every step), the per-rank GEMV `roofline`, clocks."""
    import json
    import torch.distributed as dist

    from paper_1511_07207_b200.core import SolverConfig
    from paper_1511_07207_b200.distributed import (CudaShardOps, TorchComm, cg_solve_sharded, row_partition,
                                                   spd_block_device)

    comm = TorchComm()
    ops = CudaShardOps(be.ctx)
    ops.bind_current_stream()
    stream = torch.cuda.current_stream()
    n, iters = args.n, args.iters
    G, q = comm.size, comm.rank
    n_loc, N = row_partition(n, G)
    r0, r1 = q * n_loc, min(n, (q + 1) * n_loc)
    A_blk = torch.zeros((n, n_loc), dtype=torch.float64, device=dev)
    if r1 > r0:
        A_blk[:, : r1 - r0] = spd_block_device(n, r0, r1, torch, dev)
    b = torch.zeros(n_loc, dtype=torch.float64, device=dev)
    b[: r1 - r0] = 1.0
    x0 = torch.zeros(n_loc, dtype=torch.float64, device=dev)
    cfg = SolverConfig(tolerance=1e-300, max_iterations=iters)
    for _ in range(args.warmup):
        cg_solve_sharded(A_blk, b, x0, n, cfg, comm, ops)
    torch.cuda.synchronize()
    comm.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = be.ctx.launches()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            x, rep = cg_solve_sharded(A_blk, b, x0, n, cfg, comm, ops)
        e1.record(stream)
        torch.cuda.synchronize()
    comm.barrier()
    launches = be.ctx.launches() - l0
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())

    # per-rank GEMV roofline: the local n x n_loc block streamed once (8 (n n_loc + n + n_loc) B)
    full = torch.zeros(N, dtype=torch.float64, device=dev)
    y = torch.empty(n_loc, dtype=torch.float64, device=dev)
    for _ in range(3):
        ops.gemv(A_blk, n_loc, n_loc, n, full, y)
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(20):
        ops.gemv(A_blk, n_loc, n_loc, n, full, y)
    g1.record(stream)
    torch.cuda.synchronize()
    gemv_ms = torch.tensor([g0.elapsed_time(g1) / 20], dtype=torch.float64, device=dev)
    dist.all_reduce(gemv_ms, op=dist.ReduceOp.MAX)
    gemv_ms = float(gemv_ms.item())
    hbm_peak, peak_src = _peaks()
    gbytes = 8.0 * (n * n_loc + n + n_loc)
    achieved = gbytes / (gemv_ms / 1e3) / 1e9

    # end to end: pinned host shards -> device -> solve -> x shard back, every step
    A_h = torch.empty((n, n_loc), dtype=torch.float64, pin_memory=True)
    A_h.copy_(A_blk)
    b_h = torch.empty(n_loc, dtype=torch.float64, pin_memory=True)
    b_h.copy_(b)
    x0_h = torch.zeros(n_loc, dtype=torch.float64, pin_memory=True)
    x_h = torch.empty(n_loc, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    comm.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        A_blk.copy_(A_h, non_blocking=True)
        b.copy_(b_h, non_blocking=True)
        x0.copy_(x0_h, non_blocking=True)
        x, rep = cg_solve_sharded(A_blk, b, x0, n, cfg, comm, ops)
        x_h.copy_(x, non_blocking=True)
    f1.record(stream)
    torch.cuda.synchronize()
    comm.barrier()
    e2e_ms = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    lu = bench_block_cyclic_lu(args, torch, dev, comm, ops) if not getattr(args, "only_cg", False) else None
    if q == 0:
        value = iters * args.steps / (ms / 1e3)
        unit = f"CG iters/s (n={n} fp64)"
        print(json.dumps({
            "metric": BASELINE_METRIC, "value": round(value, 3), "unit": unit, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (hash-generated symmetric A = S + 1.5 sqrt(n) I, row blocks generated per rank)",
            "config": {"workload": f"C4: CG dense SPD n={n} fp64 row-sharded over {G} GPUs, {iters} iterations/step",
                       "n": n, "iters_per_step": iters, "parallelism": f"rows{G}",
                       "l2_policy": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4), "traffic": None,
                         "kernel": "per-rank ds_gemv on the n x n_loc block (max over ranks)",
                         "algorithmic_bytes_per_launch": gbytes, "avg_launch_ms": round(gemv_ms, 4),
                         "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": {"value": iters * args.steps / (e2e_ms / 1e3), "unit": unit,
                    "h2d_bytes_per_step": int(G * (A_h.numel() + 2 * n_loc) * 8),
                    "d2h_bytes_per_step": int(G * n_loc * 8), "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": launches, "clocks": clk.summary(),
            "components": {"lu_block_cyclic": lu} if lu else {},
            "timing": "max over ranks of CUDA-event time"}), flush=True)


def bench_block_cyclic_lu(args, torch, dev, comm, ops):
    """1-D block-cyclic LU (b=64, NB-wide column blocks dealt round-robin) of a uniform
    U[-1,1] n x n matrix (every column block seeded by its index, so the matrix does not
    depend on N); GFLOP/s of 2n^3/3, max over ranks of the CUDA-event time."""
    import torch.distributed as dist

    from paper_1511_07207_b200.distributed import local_blocks, lu_factor_block_cyclic, outer_block

    n, b = args.lu_n5, 64
    G, q = comm.size, comm.rank
    NB = outer_block(b, n)
    blocks = local_blocks(-(-n // NB), q, G)
    ncols = sum(min(NB, n - k * NB) for k in blocks)

    def make():
        W = torch.empty((ncols, n), dtype=torch.float64, device=dev)
        c0 = 0
        for k in blocks:
            w = min(NB, n - k * NB)
            g = torch.Generator(device=dev)
            g.manual_seed(1000 + k)
            W[c0:c0 + w] = torch.rand((w, n), dtype=torch.float64, device=dev, generator=g).mul_(2.0).sub_(1.0)
            c0 += w
        return W

    W = make()
    lu_factor_block_cyclic(W, n, b, comm, ops)  # warm-up
    W = make()
    torch.cuda.synchronize()
    comm.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    piv, sing = lu_factor_block_cyclic(W, n, b, comm, ops)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    tf = 2.0 * n ** 3 / 3.0 / (ms / 1e3) / 1e12
    del W
    torch.cuda.empty_cache()
    return {"workload": f"1-D block-cyclic LU b=64 (NB={NB} column blocks) uniform U[-1,1] n={n} fp64 over {G} GPUs",
            "value": round(tf * 1e3, 1), "unit": "GFLOP/s", "ms": round(ms, 2), "singular": sing,
            "fp64_peak_tflops_per_gpu": 37.1, "frac_of_aggregate_fp64_peak": round(tf / (37.1 * G), 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--lu-n", type=int, default=16384)
    ap.add_argument("--lu-n5", type=int, default=32768)
    ap.add_argument("--gmres-n", type=int, default=65536)
    ap.add_argument("--only-cg", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-sharded", action="store_true", help="run the row-sharded (N>1) path even at N=1")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
