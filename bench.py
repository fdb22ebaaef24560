#!/usr/bin/env python
"""Benchmark of the B200 densolve hot path (BASELINE.json metric).

Headline (``value``): CG iterations/s on config C4, the reference's own spd recipe
(harness.py:88-91: M ~ U[-1,1] from default_rng([0, n, 2]), A = M^T M + n I, exactly
symmetric) at n=32768 fp64, generated on the device by the library's bit-identical
PCG64 stream (csrc/ds_gen.cu), A resident in HBM.  One *step* = one ``cg_solve`` call
with tolerance 1e-300 and max_iterations=ITERS (the reference's fixed-iteration idiom,
tests/test_krylov.py:188-191): symmetry gate + setup + ITERS iterations.  ``e2e`` is the
same metric through the public API with pinned HOST buffers (A, b, x0 uploaded and x
downloaded inside every step).  ``components`` adds GMRES(30) C2 and fp64 n=32768,
GMRES(50) n=65536 fp32 (C5), BiCGSTAB and Cholesky on the C4 matrix, blocked LU (b=64)
+ lu_solve at n=16384 (C3) and n=32768 (C5 per-GPU size) on the uniform recipe, each
with the reference CPU path timed beside it on this host.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--impl reference times the UNMODIFIED reference package (baseline/_ref, installed from
/root/reference with pip) through its public API -- densolve.cg_solve(A, b, x0,
SolverConfig(tolerance=1e-300, max_iterations=ITERS), get_backend("blocked")) -- on the
same matrix bytes (generated once, outside the timed region, by the same device
generator and downloaded), the same ITERS per step and the same config, on the host
cores, rank 0 only.
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
FP32_PEAK_TFLOPS = 74.4  # FFMA: 148 SMs x 128 lanes x 2 flop x 1.965 GHz (nominal at the max SM clock)
FP32_PEAK_SOURCE = "nominal: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz (not measured)"


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
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def host_info():
    """CPU model, core count, RAM and the BLAS thread pools the CPU legs run on."""
    info = {"cores": os.cpu_count() or 1}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemTotal"):
                    info["ram_gib"] = round(int(line.split()[1]) / 2 ** 20, 1)
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "threading_layer")}
                        for d in threadpool_info()]
    except Exception:  # noqa: BLE001 - informational
        pass
    return info


def ref_densolve():
    """The UNMODIFIED reference package, pip-installed from /root/reference into
    baseline/_ref (__graft_entry__.build()); it travels to the GPU box with the repo."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(p, "densolve")):
        raise ImportError(f"{p}/densolve is missing (install: see DESIGN.md §8)")
    if p not in sys.path:
        sys.path.insert(0, p)
    import densolve
    return densolve


def c4_config(n, iters, ws):
    """The workload both arms run (identical dicts: the driver compares them)."""
    return {"workload": f"C4: CG dense SPD n={n} fp64, reference spd recipe (harness.py:88-91, "
                        f"default_rng([0, n, 2])), fixed {iters} iterations per step (tolerance 1e-300)",
            "n": n, "iters_per_step": iters, "seed": 0,
            "l2_policy": f"inputs larger than L2 (A = {8 * n * n / 2 ** 30:.1f} GiB >> 126 MB L2)",
            "parallelism": f"rows{ws}"}


def c4_host_inputs(n):
    """(A, b) of config C4 on the host, the bytes the B200 arm solves: generated by the
    device generator when a GPU is present (the spd recipe's M^T M is then the DMMA SYRK),
    else by the recipe in NumPy with M.T @ M.copy() (gemm; the reference's syrk call
    crashes at n=32768)."""
    try:
        from paper_1511_07207_b200 import get_backend
        from paper_1511_07207_b200.harness import generate_problem_device
        be = get_backend("b200")
        dA, db, _ = generate_problem_device("spd", n, 0, "f64", be)
        A, b = dA.to_host(), db.to_host()
        dA.free(), db.free()
        be.ctx.synchronize()
        return A, b, "device generator (ds_generate, same bytes as the B200 arm)"
    except RuntimeError:
        rng = np.random.default_rng([0, n, 2])
        M = rng.uniform(-1.0, 1.0, size=(n, n))
        S = M.T @ M.copy() + n * np.eye(n)
        del M
        A = np.asfortranarray(np.tril(S) + np.tril(S, -1).T)
        xt = rng.uniform(-1.0, 1.0, size=n)
        return A, A @ xt, "NumPy recipe (no GPU visible)"


def ref_cg_step(densolve, A, b, x0, iters):
    cfg = densolve.SolverConfig(tolerance=1e-300, max_iterations=iters)
    be = densolve.get_backend("blocked")
    t0 = time.perf_counter()
    _, rep = densolve.cg_solve(A, b, x0, cfg, be)
    dt = time.perf_counter() - t0
    assert rep.iterations == iters, rep.iterations
    return dt


# ---------------------------------------------------------------------------- reference arm
REF_MAX_STEPS = 3  # ~43 s per 100-iteration step at n=32768 on 16 cores: the run stays near 3 min


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    n, iters = args.n, args.iters
    try:
        densolve = ref_densolve()
    except ImportError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}), flush=True)
        return
    A, b, src = c4_host_inputs(n)
    x0 = np.zeros(n)
    warm, steps = min(args.warmup, 1), max(1, min(args.steps, REF_MAX_STEPS))
    times = []
    for k in range(warm + steps):
        dt = ref_cg_step(densolve, A, b, x0, iters)
        if k >= warm:
            times.append(dt)
    tot = sum(times)
    val = iters * len(times) / tot
    info = host_info()
    unit = f"CG iters/s (n={n} fp64)"
    sample = (f"densolve.cg_solve (unmodified reference, baseline/_ref) with get_backend('blocked'), "
              f"{iters} iterations per call incl. its symmetry gate, {len(times)} timed call(s) after {warm} "
              f"warm-up; A from the {src}")
    line = {"impl": "reference", "metric": BASELINE_METRIC, "value": val, "unit": unit, "n_gpus": ws,
            "steps": len(times), "steps_requested": args.steps, "warmup": warm,
            "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": c4_config(n, iters, ws),
            "cpu_baseline": {"value": val, "unit": unit, "cores": info["cores"], "kind": "reference",
                             "sample": sample, "host": info},
            "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- B200 arm
def cpu_baseline_c4(A_h, b_h, n, iters):
    """One bounded call of the reference CG on this host on the B200 arm's own bytes."""
    info = host_info()
    try:
        densolve = ref_densolve()
        dt = ref_cg_step(densolve, A_h, b_h, np.zeros(n), iters)
        kind, what = "reference", "densolve.cg_solve (unmodified reference, baseline/_ref), get_backend('blocked')"
    except ImportError:
        from oracle import densolve_oracle as O
        t0 = time.perf_counter()
        O.cg(A_h, b_h, np.zeros(n), 1e-300, iters, O.Ops(threads=info["cores"]))
        dt = time.perf_counter() - t0
        kind, what = "port", "oracle.cg (NumPy restatement of krylov.cg_solve)"
    return {"value": iters / dt, "unit": f"CG iters/s (n={n} fp64)", "cores": info["cores"], "kind": kind,
            "sample": f"one call of {what} incl. its symmetry gate, n={n}, {iters} iterations, {dt:.1f} s, "
                      "same matrix bytes", "host": info}


def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = ws > 1 or args.force_sharded
    if ws > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=dev)
    from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend, pinned_empty
    from paper_1511_07207_b200.device import DeviceArray
    from paper_1511_07207_b200.harness import generate_problem_device

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
            return bench_sharded_cg(args, torch, dev, local)
        finally:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()

    # ---- inputs: the reference spd recipe, generated on the device (ds_generate)
    dA, db, _ = generate_problem_device("spd", n, 0, "f64", be)
    dx0 = DeviceArray(ctx, (n,), np.float64)
    ctx.lib.ds_memset(ctx.handle, dx0.ptr, 0, 8 * n)
    # host copies (pinned) for the end-to-end arm and the CPU baseline
    A_h = pinned_empty((n, n), np.float64, order="F")
    dA.to_host(out=A_h)
    b_h = pinned_empty((n,), np.float64)
    b_h[:] = db.to_host()
    x0_h = pinned_empty((n,), np.float64)
    x0_h[:] = 0.0
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
                "kernel": "ds_colstream_mv_kernel<double,2,8> + ds_colstream_reduce_kernel (ds_gemv)",
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
    del dx0  # the resident A stays for the components below
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

    cpu = None if args.no_cpu_baseline else cpu_baseline_c4(A_h, b_h, n, min(iters, 30))
    components = {}
    if not args.only_cg:
        from paper_1511_07207_b200 import bicgstab_solve, cholesky_factor
        components["bicgstab"] = bench_bicgstab(args, torch, stream, be, dA, db, dx0, n, bicgstab_solve,
                                                SolverConfig, hbm_peak, A_h, b_h)
        components["cholesky"] = bench_cholesky(args, torch, stream, be, dA, n, cholesky_factor, A_h)
    del dA, A_h
    torch.cuda.empty_cache()
    if not args.only_cg:
        components["gmres_c2"] = bench_gmres(args, torch, stream, be, 4096, 30, "f64", "C2", hbm_peak)
        components["gmres_fp64_n32768"] = bench_gmres(args, torch, stream, be, args.n, 30, "f64",
                                                      "north_star GMRES fp64", hbm_peak)
        components["gmres_c5"] = bench_gmres_c5(args, torch, dev, stream, be, hbm_peak)
        lu_fit = None if args.no_cpu_baseline else reference_lu_fit()
        components["lu_c3"] = bench_lu(args, torch, stream, be, args.lu_n, lu_fit, hbm_peak)
        components["lu_c5"] = bench_lu(args, torch, stream, be, args.lu_n5, lu_fit, hbm_peak)
        # fp32 LU (the reference's f32 families, tests/test_direct.py:123-139) at the C3 size
        lu_fit32 = None if args.no_cpu_baseline else reference_lu_fit(np.float32)
        components["lu_c3_f32"] = bench_lu(args, torch, stream, be, args.lu_n, lu_fit32, hbm_peak, "f32")

    line = {"metric": BASELINE_METRIC, "value": round(value, 3), "unit": f"CG iters/s (n={n} fp64)",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the reference's seeded spd recipe (harness.py:88-91) generated on the device "
                    "(ds_generate: bit-identical PCG64 stream, M^T M by the DMMA SYRK)",
            "config": c4_config(n, iters, ws),
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


def _gmres_cycle_bytes(n, m, s):
    """Algorithmic bytes of one GMRES(m) cycle: (m + 2) passes over A (m Arnoldi GEMVs +
    residual + true residual), per step k the basis traffic (2k + 7) n, and the x update."""
    return s * ((m + 2) * n * n + sum((2 * k + 7) * n for k in range(m)) + (m + 2) * n)


def _ref_gmres_cycle(A, b, m, reps=1):
    """Seconds of one full GMRES(m) cycle of the unmodified reference (best of reps)."""
    densolve = ref_densolve()
    cfg = densolve.SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
    be = densolve.get_backend("blocked")
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        _, rep = densolve.gmres_solve(A, b, np.zeros_like(b), cfg, be)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, rep.iterations


def bench_gmres(args, torch, stream, be, n, m, prec, tag, hbm_peak):
    """GMRES(m) on the reference general_nonsymmetric recipe (harness.py:92-98), one full cycle
    per step (residual + m Arnoldi steps + update + true residual)."""
    from paper_1511_07207_b200 import SolverConfig, gmres_solve
    from paper_1511_07207_b200.harness import generate_problem_device

    dA, db, _ = generate_problem_device("general_nonsymmetric", n, 0, prec, be)
    dx0 = be.stage_in(np.zeros(n, dtype=dA.dtype))
    cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
    ms, (x, rep) = _timed(torch, stream, lambda: gmres_solve(dA, db, dx0, cfg, be), 10 if n <= 8192 else 3)
    s = dA.dtype.itemsize
    gbs = _gmres_cycle_bytes(n, m, s) / (ms / 1e3) / 1e9
    out = {"workload": f"{tag}: GMRES({m}) general_nonsymmetric recipe n={n} {prec}, one full cycle per step",
           "value": round(rep.iterations / (ms / 1e3), 1), "unit": "inner iters/s", "ms_per_step": round(ms, 4),
           "iterations": rep.iterations, "GBps": round(gbs, 1), "frac_of_hbm_peak": round(gbs / hbm_peak, 4)}
    if not args.no_cpu_baseline:
        A, b = dA.to_host(), db.to_host()
        del dA
        dt, its = _ref_gmres_cycle(A, b, m, reps=3 if n <= 8192 else 1)
        out["cpu_baseline"] = {"value": round(its / dt, 2), "unit": "inner iters/s", "cores": os.cpu_count(),
                               "kind": "reference",
                               "sample": f"one cycle of densolve.gmres_solve (baseline/_ref, 'blocked'), same bytes, "
                                         f"{dt:.2f} s"}
    torch.cuda.empty_cache()
    return out


def bench_gmres_c5(args, torch, dev, stream, be, hbm_peak):
    """C5: GMRES(50) n=65536 fp32, one full cycle per step (HBM-capacity sizing, 1 GPU).
    Matrix: the uniform recipe's stream (default_rng([3, n, 1]), ds_generate) shifted by
    1.5 sqrt(n) I.  The reference general_nonsymmetric recipe contracts ~300x per step, so a
    FIXED 50-step cycle underflows the fp32 Givens estimate after ~16 steps; the shifted
    uniform matrix (circular-law spectrum, ~0.38 per step) keeps every step meaningful.
    (Parity on the general_nonsymmetric recipe itself: tests/test_gpu_config_parity.py.)"""
    from paper_1511_07207_b200 import SolverConfig, gmres_solve
    from paper_1511_07207_b200.harness import generate_problem_device

    n, m = args.gmres_n, 50
    dA, db, dxt = generate_problem_device("uniform", n, 3, "f32", be)
    tA = torch.as_tensor(dA, device=dev)
    torch.cuda.synchronize()
    tA.diagonal().add_(1.5 * float(n) ** 0.5)
    torch.cuda.synchronize()
    from ctypes import c_void_p
    from paper_1511_07207_b200 import _lib
    _lib.check(be.ctx.lib.ds_gemv(be.ctx.handle, _lib.DS_F32, n, n, c_void_p(dA.ptr), dA.ld,
                                  c_void_p(dxt.ptr), c_void_p(db.ptr)))  # b = A x_true (library GEMV)
    dx0 = be.stage_in(np.zeros(n, dtype=np.float32))
    cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
    ms, (x, rep) = _timed(torch, stream, lambda: gmres_solve(dA, db, dx0, cfg, be), 3)
    gbs = _gmres_cycle_bytes(n, m, 4.0) / (ms / 1e3) / 1e9
    out = {"workload": f"C5: GMRES({m}) dense nonsymmetric n={n} fp32, uniform recipe + 1.5 sqrt(n) I "
                       "(device-generated), one full cycle per step", "cycles": len(rep.restart_cycles or []),
           "iterations": rep.iterations, "value": round(rep.iterations / (ms / 1e3), 1), "unit": "inner iters/s",
           "ms_per_step": round(ms, 3), "GBps": round(gbs, 1), "frac_of_hbm_peak": round(gbs / hbm_peak, 4)}
    if not args.no_cpu_baseline:
        A, b = dA.to_host(), db.to_host()
        del tA, dA
        dt, its = _ref_gmres_cycle(A, b, m)
        out["cpu_baseline"] = {"value": round(its / dt, 2), "unit": "inner iters/s", "cores": os.cpu_count(),
                               "kind": "reference",
                               "sample": f"one 50-step cycle of densolve.gmres_solve (baseline/_ref, 'blocked'), "
                                         f"same bytes, {dt:.1f} s"}
        del A
    torch.cuda.empty_cache()
    return out


def bench_bicgstab(args, torch, stream, be, dA, db, dx0, n, bicgstab_solve, SolverConfig, hbm_peak, A_h, b_h):
    """BiCGSTAB on the C4 matrix, fixed 50 iterations per step."""
    iters = 50
    cfg = SolverConfig(tolerance=1e-300, max_iterations=iters)
    ms, (x, rep) = _timed(torch, stream, lambda: bicgstab_solve(dA, db, dx0, cfg, be), 2)
    its = rep.iterations
    gbs = 8.0 * (2 * its + 1) * (n * n) / (ms / 1e3) / 1e9
    out = {"workload": f"BiCGSTAB dense SPD n={n} fp64 (C4 matrix), fixed {iters} iterations per step",
           "value": round(its / (ms / 1e3), 2), "unit": "iters/s", "ms_per_step": round(ms, 3),
           "iterations": its, "breakdown": rep.breakdown, "GBps_A_stream": round(gbs, 1),
           "frac_of_hbm_peak": round(gbs / hbm_peak, 4)}
    if not args.no_cpu_baseline:
        densolve = ref_densolve()
        k = 10
        t0 = time.perf_counter()
        _, r = densolve.bicgstab_solve(A_h, b_h, np.zeros(n), densolve.SolverConfig(tolerance=1e-300,
                                       max_iterations=k), densolve.get_backend("blocked"))
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": round(r.iterations / dt, 3), "unit": "iters/s", "cores": os.cpu_count(),
                               "kind": "reference",
                               "sample": f"densolve.bicgstab_solve (baseline/_ref), {r.iterations} iterations, {dt:.1f} s"}
    return out


def bench_cholesky(args, torch, stream, be, dA, n, cholesky_factor, A_h=None):
    """Cholesky of the C4 SPD matrix, b=64, device-resident.  CPU
    baseline: the reference cholesky_factor (b=64, 'blocked') at n = 2048 / 4096 on the spd
    recipe fitted to t = a n^3 (labelled extrapolated), plus scipy's LAPACK dpotrf at full n
    on the same bytes as a labelled comparator."""
    runs = [_timed(torch, stream, lambda: cholesky_factor(dA, 64, be), 1)[0] for _ in range(3)]
    ms = min(runs)  # 1 warm-up (inside _timed) + best of 3, harness.py:281-294
    tf = n ** 3 / 3.0 / (ms / 1e3) / 1e12
    out = {"workload": f"blocked Cholesky b=64, dense SPD n={n} fp64 (C4 matrix), device-resident; best of 3",
           "value": round(tf * 1e3, 1), "unit": "GFLOP/s", "ms": round(ms, 2),
           "ms_runs": [round(r, 2) for r in runs],
           "fp64_peak_tflops": FP64_PEAK_TFLOPS, "frac_of_fp64_peak": round(tf / FP64_PEAK_TFLOPS, 4)}
    if args.no_cpu_baseline:
        return out
    try:
        from paper_1511_07207_b200.harness import ProblemSpec, generate_problem
        densolve = ref_densolve()
        rbe = densolve.get_backend("blocked")
        pts = []
        for m in (2048, 4096):
            S, _, _ = generate_problem(ProblemSpec(kind="spd", n=m, seed=0))
            t0 = time.perf_counter()
            densolve.cholesky_factor(S, 64, rbe)
            pts.append((m, time.perf_counter() - t0))
        a = sum(t * m ** 3 for m, t in pts) / sum(m ** 6 for m, _ in pts)
        te = a * n ** 3
        cpu = {"value": round(n ** 3 / 3.0 / te / 1e9, 3), "unit": "GFLOP/s", "cores": host_info()["cores"],
               "kind": "reference",
               "sample": f"EXTRAPOLATED: densolve.cholesky_factor (baseline/_ref, b=64, 'blocked') timed at "
                         f"n=2048/4096, t = a n^3 -> {te:.0f} s at n={n}",
               "points": [{"n": m, "s": round(t, 3), "GFLOP/s": round(m ** 3 / 3 / t / 1e9, 3)} for m, t in pts]}
        if A_h is not None:
            import scipy.linalg
            t0 = time.perf_counter()
            scipy.linalg.cholesky(A_h, lower=True, overwrite_a=False, check_finite=False)
            tl = time.perf_counter() - t0
            cpu["lapack_comparator"] = {"value": round(n ** 3 / 3.0 / tl / 1e9, 1), "unit": "GFLOP/s",
                                        "s": round(tl, 2),
                                        "what": "scipy.linalg.cholesky (LAPACK dpotrf, OpenBLAS) at full n on the "
                                                "same bytes; NOT the reference"}
        out["cpu_baseline"] = cpu
    except Exception as e:  # the reference install is optional on the box
        out["cpu_baseline"] = {"unavailable": str(e)[:200]}
    return out


def reference_lu_fit(dtype=np.float64):
    """The reference lu_factor_blocked (b=64, 'blocked' backend, all cores) on the uniform
    recipe at n = 2048 and 4096, fitted to t = a n^3 (full n needs hours)."""
    from paper_1511_07207_b200.harness import generate_uniform
    densolve = ref_densolve()
    be = densolve.get_backend("blocked")
    pts = []
    for n in (2048, 4096):
        A, _, _ = generate_uniform(n, 1)
        A = np.asfortranarray(A, dtype=dtype)
        t0 = time.perf_counter()
        densolve.lu_factor_blocked(A, 64, be)
        pts.append((n, time.perf_counter() - t0))
    a = sum(t * n ** 3 for n, t in pts) / sum(n ** 6 for n, _ in pts)  # least squares through 0
    return {"a": a, "points": [{"n": n, "s": round(t, 3), "GFLOP/s": round(2 * n ** 3 / 3 / t / 1e9, 3)}
                               for n, t in pts]}


def bench_lu(args, torch, stream, be, n, lu_fit, hbm_peak, prec="f64"):
    """Blocked LU b=64 on the uniform recipe (C3 pivoting family, default_rng([1, n, 1]),
    ds_generate) + lu_solve of b = A x_true; CPU: the reference extrapolated from n=2048/4096
    and LAPACK getrf (scipy) at full n as a labelled comparator."""
    from paper_1511_07207_b200 import lu_factor_blocked, lu_solve
    from paper_1511_07207_b200.harness import generate_problem_device

    dA, db, dxt = generate_problem_device("uniform", n, 1, prec, be)
    esize = 8 if prec == "f64" else 4
    torch.cuda.synchronize()
    f = lu_factor_blocked(dA, 64, be)  # warm-up
    del f
    # 1 warm-up + best-of-3, the reference's own timing protocol (harness.py:281-294)
    runs = [_timed(torch, stream, lambda: lu_factor_blocked(dA, 64, be), 1)[0] for _ in range(3)]
    ms = min(runs)
    f = lu_factor_blocked(dA, 64, be)
    sms, x = _timed(torch, stream, lambda: lu_solve(f, db), 5)
    err = float(np.max(np.abs(x.to_host() - dxt.to_host())))
    sbytes = float(esize) * n * n  # one pass over each triangle of the packed factors
    flops = 2.0 * n ** 3 / 3.0
    tf = flops / (ms / 1e3) / 1e12
    out = {"workload": f"blocked LU b=64, uniform recipe n={n} {'fp64' if prec == 'f64' else 'fp32'} "
                       "(pivoting family), device-resident (includes the device copy of A, direct.py:61); "
                       "best of 3 after 1 warm-up",
           "value": round(tf * 1e3, 1), "unit": "GFLOP/s", "ms": round(ms, 2), "ms_runs": [round(r, 2) for r in runs]}
    if prec == "f64":
        out.update({"fp64_peak_tflops": FP64_PEAK_TFLOPS, "frac_of_fp64_peak": round(tf / FP64_PEAK_TFLOPS, 4)})
    else:  # FFMA on the CUDA cores (no FP32 tensor-core GEMM that keeps fp32 rounding)
        out.update({"fp32_peak_tflops": FP32_PEAK_TFLOPS, "fp32_peak_source": FP32_PEAK_SOURCE,
                    "frac_of_fp32_peak": round(tf / FP32_PEAK_TFLOPS, 4)})
    out.update({
           "lu_solve": {"ms": round(sms, 4), "GBps": round(sbytes / (sms / 1e3) / 1e9, 1),
                        "frac_of_hbm_peak": round(sbytes / (sms / 1e3) / 1e9 / hbm_peak, 4),
                        "algorithmic_bytes": sbytes, "max_abs_err_vs_x_true": err}})
    del f
    if lu_fit is not None:
        import scipy.linalg
        A = dA.to_host()
        del dA
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        scipy.linalg.lu_factor(A, overwrite_a=True, check_finite=False)
        tl = time.perf_counter() - t0
        del A
        te = lu_fit["a"] * n ** 3
        out["cpu_baseline"] = {"value": round(flops / te / 1e9, 3), "unit": "GFLOP/s", "cores": os.cpu_count(),
                               "kind": "reference",
                               "sample": f"EXTRAPOLATED: densolve.lu_factor_blocked (baseline/_ref, b=64, 'blocked') "
                                         f"timed at n=2048/4096, t = a n^3 -> {te:.0f} s at n={n}",
                               "points": lu_fit["points"],
                               "lapack_comparator": {"value": round(flops / tl / 1e9, 1), "unit": "GFLOP/s",
                                                     "s": round(tl, 2),
                                                     "what": f"scipy.linalg.lu_factor (LAPACK {'d' if prec == 'f64' else 's'}getrf, OpenBLAS) at "
                                                             "full n on the same bytes; NOT the reference"}}
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------- N > 1 (torchrun)
def bench_sharded_cg(args, torch, dev, local):
    """C4 CG row-sharded through the public API: `get_backend("b200", distributed=True)` under
    torchrun (one process per GPU, exchange regions mapped through CUDA IPC), or
    `get_backend("b200", devices=[0])` for `--force-sharded` at N=1.  The whole iteration
    loop runs in the library (ds_cg_sharded: the all-gathers of p and of the reduction
    records are fused into the producing kernels over peer memory).  Same JSON contract as
    the 1-GPU line: device-resident `value` (max over ranks of the CUDA-event time), `e2e`
    (each rank uploads its row block of A, b, x0 from pinned host memory and gathers the
    whole x every step), the per-rank GEMV `roofline`, clocks."""
    import json
    import torch.distributed as dist

    from paper_1511_07207_b200 import SolverConfig, cg_solve, get_backend, pinned_empty
    from paper_1511_07207_b200.device import DeviceArray, _padded_ld
    from paper_1511_07207_b200.harness import generate_problem_device
    from paper_1511_07207_b200.sharded import ShardedMatrix, ShardedVector

    multi = dist.is_initialized()
    be = get_backend("b200", distributed=True, device=local) if multi else get_backend("b200", devices=[local])
    G, q = be.nshards, be.local_ranks[0]
    sctx = be.shard_contexts[0]
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sctx.set_stream(stream.cuda_stream)  # the shard's library work on this stream: the events see it
    n, iters = args.n, args.iters
    ss = be.shardset(n, np.float64)
    r0, r1 = ss.rows(q)
    n_loc = ss.n_loc
    # every rank generates the full C4 matrix (the reference spd recipe, same bytes as the
    # 1-GPU arm) and keeps its row block
    gen = get_backend("b200", device=local)
    dA, db, _ = generate_problem_device("spd", n, 0, "f64", gen)
    gen.ctx.synchronize()
    blk = DeviceArray(sctx, (n_loc, n), np.float64, ld=_padded_ld(n_loc))
    bpart = DeviceArray(sctx, (n_loc,), np.float64)
    x0part = DeviceArray(sctx, (n_loc,), np.float64)
    tA, tb = torch.as_tensor(dA, device=dev), torch.as_tensor(db, device=dev)
    tblk, tbp = torch.as_tensor(blk, device=dev), torch.as_tensor(bpart, device=dev)
    tblk.zero_()
    tbp.zero_()
    torch.as_tensor(x0part, device=dev).zero_()
    if r1 > r0:
        tblk[: r1 - r0].copy_(tA[r0:r1, :])
        tbp[: r1 - r0].copy_(tb[r0:r1])
    torch.cuda.synchronize()
    del tA, tb, tblk, tbp, dA, db
    A_sh, b_sh, x0_sh = ShardedMatrix(ss, [blk]), ShardedVector(ss, [bpart]), ShardedVector(ss, [x0part])
    cfg = SolverConfig(tolerance=1e-300, max_iterations=iters)

    def max_over_ranks(v):
        if not multi:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if multi:
            dist.barrier()

    for _ in range(args.warmup):
        cg_solve(A_sh, b_sh, x0_sh, cfg, be)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = sctx.launches()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            x, rep = cg_solve(A_sh, b_sh, x0_sh, cfg, be)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    assert rep.iterations == iters
    launches = sctx.launches() - l0
    ms = max_over_ranks(e0.elapsed_time(e1))

    # per-rank GEMV roofline: the local n_loc x n block streamed once (8 (n n_loc + n + n_loc) B)
    from ctypes import c_void_p

    from paper_1511_07207_b200 import _lib
    xin = DeviceArray(sctx, (n,), np.float64)
    torch.as_tensor(xin, device=dev).fill_(1.0)
    y = DeviceArray(sctx, (n_loc,), np.float64)

    def gemv():
        _lib.check(sctx.lib.ds_gemv(sctx.handle, _lib.DS_F64, n_loc, n, c_void_p(blk.ptr), blk.ld,
                                    c_void_p(xin.ptr), c_void_p(y.ptr)))

    for _ in range(3):
        gemv()
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(20):
        gemv()
    g1.record(stream)
    torch.cuda.synchronize()
    gemv_ms = max_over_ranks(g0.elapsed_time(g1) / 20)
    hbm_peak, peak_src = _peaks()
    gbytes = 8.0 * (n * n_loc + n + n_loc)
    achieved = gbytes / (gemv_ms / 1e3) / 1e9

    # end to end: pinned host row block, b and x0 shards -> device -> solve -> whole x back
    A_h = pinned_empty((n_loc, n), np.float64, order="F")
    blk.to_host(out=A_h)
    b_h = pinned_empty((n_loc,), np.float64)
    bpart.to_host(out=b_h)
    x0_h = pinned_empty((n_loc,), np.float64)
    x0_h[:] = 0.0
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        blk.upload(A_h)
        bpart.upload(b_h)
        x0part.upload(x0_h)
        xs, rep = cg_solve(A_sh, b_sh, x0_sh, cfg, be)
        x_full = xs.to_host()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(max(f0.elapsed_time(f1), 1e3 * (time.perf_counter() - t0)))
    barrier()
    lu = None
    if multi and not getattr(args, "only_cg", False):
        lu = bench_block_cyclic_lu(args, torch, dev, be)
    if q == 0:
        value = iters * args.steps / (ms / 1e3)
        unit = f"CG iters/s (n={n} fp64)"
        print(json.dumps({
            "metric": BASELINE_METRIC, "value": round(value, 3), "unit": unit, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the reference's seeded spd recipe (harness.py:88-91) generated on the device "
                    "(ds_generate), each rank keeping its row block",
            "config": dict(c4_config(n, iters, G), api="get_backend('b200', %s)" % (
                "distributed=True" if multi else f"devices=[{local}]")),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4), "traffic": None,
                         "kernel": "per-rank ds_gemv on the n_loc x n row block (max over ranks)",
                         "algorithmic_bytes_per_launch": gbytes, "avg_launch_ms": round(gemv_ms, 4),
                         "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": {"value": iters * args.steps / (e2e_ms / 1e3), "unit": unit,
                    "h2d_bytes_per_step": int(G * (A_h.nbytes + b_h.nbytes + x0_h.nbytes)),
                    "d2h_bytes_per_step": int(G * x_full.nbytes), "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": launches, "clocks": clk.summary(),
            "components": {"lu_block_cyclic": lu} if lu else {},
            "timing": "max over ranks of CUDA-event time"}), flush=True)


def bench_block_cyclic_lu(args, torch, dev, be):
    """1-D block-cyclic LU (b=64, NB-wide column blocks dealt round-robin) of a uniform
    U[-1,1] n x n matrix (every column block seeded by its index, so the matrix does not
    depend on N), factored in the library (ds_lu_block_cyclic: panels broadcast over peer
    memory); GFLOP/s of 2n^3/3, max over ranks of the CUDA-event time."""
    import torch.distributed as dist

    from paper_1511_07207_b200.device import DeviceArray, _padded_ld
    from paper_1511_07207_b200.distributed import local_blocks, outer_block
    from paper_1511_07207_b200.sharded import lu_block_cyclic_device

    n, b = args.lu_n5, 64
    G, q = be.nshards, be.local_ranks[0]
    NB = outer_block(b, n)
    blocks = local_blocks(-(-n // NB), q, G)
    ncols = sum(min(NB, n - k * NB) for k in blocks)
    sctx = be.shard_contexts[0]
    W = DeviceArray(sctx, (n, max(ncols, 1)), np.float64, ld=_padded_ld(n))
    tW = torch.as_tensor(W, device=dev)  # (n, ncols) view, column-major

    def make():
        c0 = 0
        for k in blocks:
            w = min(NB, n - k * NB)
            g = torch.Generator(device=dev)
            g.manual_seed(1000 + k)
            tW[:, c0:c0 + w] = torch.rand((w, n), dtype=torch.float64, device=dev, generator=g).mul_(2.0).sub_(1.0).t()
            c0 += w
        torch.cuda.synchronize()

    make()
    lu_block_cyclic_device(be, [W], n, b, np.float64)  # warm-up
    make()
    dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    piv, sing = lu_block_cyclic_device(be, [W], n, b, np.float64)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    tf = 2.0 * n ** 3 / 3.0 / (ms / 1e3) / 1e12
    del tW, W
    torch.cuda.empty_cache()
    return {"workload": f"1-D block-cyclic LU b=64 (NB={NB} column blocks) uniform U[-1,1] n={n} fp64 over {G} GPUs "
                        "(ds_lu_block_cyclic, device-resident)",
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
