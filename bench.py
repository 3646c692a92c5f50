#!/usr/bin/env python
"""bench.py -- batched RVE condensation + macro solve on B200 (arXiv 2312.12771 hot path).

A step is one pass of the whole hot path over one synthetic batch (SURVEY.md
§8(a)): hom_condense (K1 assembly + K2-K4 fused Cholesky / influence solves /
Schur epilogue, all RVEs), hom_macro_solve (K5 assembly + K6/K7 PCG) and
hom_recover_fluctuations (K8).  For config 5 a step is one monolithic Newton
iteration (kinematics, condensation, residual norms, macro solve, update).

Default workload: BASELINE.json configs[2] (config 3: 64x64 macro Q1, 16384 RVEs of
32x32 Q1 with per-RVE random phases and moduli) -- the largest configuration that fits one
GPU, which is the headline when BASELINE's metric names no configuration; dense blocked
factorisation through the chunked path (four wave-aligned passes of 4144 RVEs over a 96 GB K_ff pool).
Companion keys: config 2 and config 5 (the configs whose k_condense sits furthest below
the FP64 roofline), the tile-sparse factorisation of the same workload, and the K6 SpMV
roofline on a scaled macro mesh.  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Multi-GPU (torchrun): every rank solves its own independent replica of the
workload (weak scaling, no data-path collective -- DESIGN.md §7); the timed
region is bracketed by barriers and the max over ranks is reported.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.15  # measured DMMA peak, tools/fp64_peaks.cu -> MEASURED_FP64.json / profiles/r01_fp64_peaks.txt
METRIC = "condensed RVE tangents/sec"


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def fp64_peak():
    m = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    if "fp64_tflops" in m:
        return float(m["fp64_tflops"]), "MEASURED_PEAKS.json fp64_tflops"
    f = load_json(os.path.join(ROOT, "MEASURED_FP64.json")) or {}
    if "fp64_dmma_tflops_microbench" in f:
        return float(f["fp64_dmma_tflops_microbench"]), "MEASURED_FP64.json (DMMA microbenchmark, this pool's B200)"
    return FP64_PEAK_TFLOPS, "measured DMMA microbenchmark (profiles/r01_fp64_peaks.txt)"


def dgemm_live_tflops(n: int = 8192, reps: int = 10):
    """cuBLAS DGEMM n^3 on this GPU in this run (best of `reps`, CUDA events): the second FP64
    denominator next to the DMMA microbenchmark peak."""
    import torch
    a = torch.rand(n, n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b, c
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle baseline
def oracle_step_time(wl, target_s: float = 10.0):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload and scale to one step.

    The oracle condenses `n` RVEs (phase rows replicated per RVE so nothing is deduplicated),
    then the direct macro solve runs once at full size.  Returns (seconds per full step, detail)."""
    import numpy as np

    import oracle
    nthreads = oracle.default_threads()
    per = 1 if wl.phase.shape[0] == 1 else None

    def sample(n, threads=None):
        ids = np.arange(n) % wl.n_rve
        ph = np.repeat(wl.phase, n, 0) if per else wl.phase[ids]
        mt = np.repeat(wl.mat, n, 0) if wl.mat.shape[0] == 1 else wl.mat[ids]
        t0 = time.perf_counter()
        if wl.kind == "linear":
            C = oracle.condense_batch_linear(wl.dim, wl.r, ph, mt, n, want_W=True, nthreads=threads or nthreads)[0]
        else:
            F = np.tile([1.0, 0.0, 0.0, 1.0], (n, 1))
            C = oracle.condense_batch_nh(wl.r, ph, mt, F, nthreads=threads or nthreads)["A_eff"]
        return time.perf_counter() - t0, C

    n = max(nthreads, 8)
    t, C = sample(n)
    # grow the sample to ~target_s of CPU work (RVEs repeat cyclically past n_rve, never deduplicated)
    while t < 0.6 * target_s and n < 256 * wl.n_rve:
        n = min(256 * wl.n_rve, max(n * 2, int(n * 0.8 * target_s / max(t, 1e-3))))
        t, C = sample(n)
    t_rve = t / n
    # per-core rate: one thread on a fixed 64-RVE slice
    n1 = min(64, wl.n_rve)
    t1, _ = sample(n1, threads=1)
    # macro direct solve at full size with representative tangents
    Cm = np.broadcast_to(C[:1], (wl.n_rve,) + C.shape[1:]).copy()
    t0 = time.perf_counter()
    if wl.kind == "linear":
        u = oracle.macro_solve(wl.dim, wl.nel, Cm, wl.dir_dof, wl.dir_val, body=wl.body)
        oracle.macro_kin(wl.dim, wl.nel, u)
    else:
        oracle.macro_solve(2, wl.nel, Cm, wl.dir_dof, np.zeros(len(wl.dir_dof)), S=np.zeros((wl.n_rve, 4)),
                           body=wl.body, kind=1)
    t_macro = time.perf_counter() - t0
    step = t_rve * wl.n_rve + t_macro
    what = (f"{n} of {wl.n_rve} RVEs" if n <= wl.n_rve else
            f"{n} RVE condensations (the {wl.n_rve} RVEs of the step, cyclically)")
    detail = {"cores": nthreads, "sample": f"{what} condensed (skyline Cholesky, unit-strain route, "
                                             f"{t:.1f} s) + 1 full-size direct macro solve ({t_macro:.2f} s); "
                                             f"scaled to a full step", "t_rve_s": t_rve, "t_macro_s": t_macro,
              "per_core_tangents_s": n1 / t1, "per_core_sample": f"{n1} RVEs on 1 thread ({t1:.2f} s)"}
    return step, detail


def oracle_full_steps(wl, steps: int, budget_s: float = 150.0):
    """The reference arm: full oracle steps (every RVE condensed, direct macro solve, recovery of
    every RVE), as it stands, on all host threads; stops early once `budget_s` is spent (at least one
    full step).  Returns (list of per-step seconds, cores)."""
    import numpy as np

    import oracle
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        if wl.kind == "linear":
            o = oracle.solve_linear(wl)
            oracle.recover_linear(o["W"], o["eps"])
        else:  # one monolithic Newton iteration at the reference state (the per-iteration work)
            oracle.newton_step_nh(wl, np.zeros(wl.n_dof), np.zeros((wl.n_rve, wl.n_pad)),
                                  wl.dir_val / wl.n_steps)
        times.append(time.perf_counter() - t0)
        if sum(times) > budget_s:
            break
    return times, oracle.default_threads()


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- scaled SpMV
def spmv_scaled(C_tile, nel: int = 2048, reps: int = 20):
    """K6 SpMV roofline on a scaled macro mesh (the config macro matrices are L2-resident, so the
    HBM-bound SpMV is measured on a 2-D nel x nel Q1 mesh): assemble K from C_eff tiled over all
    macro qps, then time reps launches of y = K_FF x with CUDA events on the launching stream."""
    import torch

    from paper_2312_12771_b200 import workloads as W
    from paper_2312_12771_b200.hom import Homogenizer
    t0 = time.perf_counter()
    wl = W.config2(nel=nel, r=2)
    h = Homogenizer.from_workload(wl, rve_range=(0, 4), check_info=False)  # one element's RVEs condensed
    t_setup = time.perf_counter() - t0
    C = C_tile[:1].expand(wl.n_rve, -1, -1).contiguous()
    h.macro_assemble(C)
    g = torch.Generator(device="cuda").manual_seed(12771)
    x = torch.rand(wl.n_dof, dtype=torch.float64, device="cuda", generator=g)
    x[torch.as_tensor(wl.dir_dof, device="cuda", dtype=torch.long)] = 0.0
    y = h.empty(wl.n_dof)
    for _ in range(3):
        h.macro_spmv(x, y)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        h.macro_spmv(x, y)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nnz, n = h.sizes.macro_nnz, wl.n_dof
    algo = nnz * 12 + n * (4 + 8 + 8 + 1)  # CSR values + columns, rowptr, y, x (gathered once, L2), Dirichlet mask
    peak = (load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}).get("hbm_gbs", 6447.8)
    out = {"kernel": "k_spmv (K6, 4 lanes per CSR row, batched loads)", "macro_mesh": f"{nel}x{nel} Q1", "macro_dof": n, "nnz": nnz,
           "ms_per_launch": ms, "bytes_per_launch": algo, "GBps": algo / (ms * 1e-3) / 1e9,
           "peak_GBps": peak, "frac": algo / (ms * 1e-3) / 1e9 / peak, "setup_s": t_setup,
           "values": "config-2 C_eff tiled over all macro Gauss points"}
    h.close()
    return out


# ----------------------------------------------------------------------------- tile-sparse companion
def tile_sparse_line(wl, C_dense, steps: int, warmup: int, ordering="folded"):
    """The same linear step with the tile-sparse factorisation: tangents/s and the
    k_condense roofline on the executed tile-structure flops, plus the bitwise check against the
    dense tangents of the main line (every skipped product is an exact zero)."""
    import torch

    from paper_2312_12771_b200.hom import Homogenizer
    h = Homogenizer.from_workload(wl, tile_sparse=True, rve_ordering=ordering)
    C = h.empty(h.n_rve, h.m, h.m)
    u = h.empty(h.n_dof)
    w = h.empty(h.n_rve, h.n_pad)

    def step():
        h.condense(None, C)
        h.macro_solve(C, None, 1.0, u)
        h.recover(u, w)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    h.profile(True)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof = h.profile_read()
    h.profile(False)
    cond_ms = prof["condense"][0]
    achieved = h.work.flop_executed * h.sizes.rve_count * steps / (cond_ms * 1e-3) / 1e12
    peak, _ = fp64_peak()
    out = {"value": wl.n_rve * steps / (ms * 1e-3), "unit": "tangents/s", "ms_per_step": ms / steps,
           "condense_ms_per_step": cond_ms / steps,
           "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak,
                        "algorithmic": f"{h.work.flop_executed:.4g} executed DMMA flop/RVE ({h.work.g_tiles} tiles)"},
           "bitwise_equal_to_dense": bool(torch.equal(C, C_dense))}
    h.close()
    return out


# ----------------------------------------------------------------------------- companion configs
def companion_line(cfg: int, steps: int, warmup: int):
    """Config `cfg` on its own context in the same run: tangents/s of the step and the k_condense
    roofline (dense algorithmic flops / the kernel's CUDA-event time)."""
    import torch

    from paper_2312_12771_b200 import workloads as W
    from paper_2312_12771_b200.hom import Homogenizer
    wl = W.make(cfg)
    h = Homogenizer.from_workload(wl)
    B, m = h.n_rve, h.m
    C, u, w = h.empty(B, m, m), h.empty(h.n_dof), h.empty(B, h.n_pad)
    if h.finite:
        F, Pe, Pa, du = h.empty(B, m), h.empty(B, m), h.empty(B, m), h.empty(h.n_dof)
        u0, _ = h.newton(1, tol=1e-9)  # a mid-load state
        u.copy_(u0)

    def step():
        if h.finite:
            h.macro_kinematics(u, F)
            h.condense(F, C, Pe, Pa)
            h.macro_residual_norm(Pa)
            h.micro_residual_max()
            h.macro_solve(C, Pe, scale=0.0, x=du)
            h.newton_update(u, du)
        else:
            h.condense(None, C)
            h.macro_solve(C, None, 1.0, u)
            h.recover(u, w)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    h.profile(True)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof = h.profile_read()
    h.profile(False)
    cond_ms = prof["condense"][0]
    achieved = wl.flop_per_rve() * B * steps / (cond_ms * 1e-3) / 1e12
    peak, _ = fp64_peak()
    out = {"workload": f"{wl.name}: {wl.description}", "step": "one Newton iteration" if h.finite else
           "condense + macro solve + recovery", "value": B * steps / (ms * 1e-3), "unit": "tangents/s",
           "ms_per_step": ms / steps, "condense_ms_per_step": cond_ms / steps,
           "roofline": {"bound": "tensor", "kernel": "k_condense", "achieved": achieved, "peak": peak,
                        "unit": "TFLOP/s", "frac": achieved / peak,
                        "algorithmic": f"{wl.flop_per_rve():.4g} flop/RVE x {B} RVEs per step"},
           "assembly_ms_per_step": prof["rve_assemble"][0] / steps,
           "macro_solve_ms_per_step": (prof["macro_assemble"][0] + prof["cg"][0]) / steps}
    h.close()
    return out


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-companions", action="store_true", help="skip the config-2 / config-5 companion keys")
    ap.add_argument("--sharded", action="store_true",
                    help="run the RVE-sharded multi-GPU path (NCCL process group, packed all-gather) even at N = 1 "
                         "(exercises the --gpus N code path on one GPU)")
    ap.add_argument("--spmv-nel", type=int, default=2048, help="scaled macro mesh of the K6 SpMV roofline (0: skip)")
    ap.add_argument("--macro-basis", default="dirac", choices=["dirac", "constant"],
                    help="constant: one RVE per macro element (SURVEY §8(f) 2, small strain)")
    ap.add_argument("--tile-sparse", action="store_true",
                    help="factor only the symbolic tile fill of K_ff (SURVEY §8(f) 3) instead of every lower tile")
    ap.add_argument("--macro-precond", default="auto", choices=["auto", "two_level", "jacobi"],
                    help="macro PCG preconditioner (hom_options.macro_precond; auto: two-level unless a "
                         "quarter or more of the macro DOFs are prescribed)")
    ap.add_argument("--rve-ordering", default="folded", choices=["folded", "natural"],
                    help="internal order of the RVE nodes (rows of K_ff); w at the API is natural either way")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2312_12771_b200 import workloads as W
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = W.make(args.config)
    if world > 1:  # weak scaling: one macro problem, its RVEs sharded; ~the same RVE count per GPU
        nel1 = wl.nel
        wl = W.make(args.config, nel=int(round(nel1 * world ** (1.0 / wl.dim))))
    n_rve_run = wl.n_rve // wl.n_qp if args.macro_basis == "constant" else wl.n_rve  # one RVE per element
    config = {"workload": f"{wl.name}: {wl.description}", "config_index": args.config,
              "n_rve": n_rve_run, "rve_dofs": wl.n_pad, "n_f": wl.n_f, "macro_dof": wl.n_dof,
              "flop_per_rve": wl.flop_per_rve(),
              "parallelism": (f"rve-sharded x{world} (packed C_eff all-gather, replicated macro CG)"
                              if world > 1 or args.sharded else "single"),
              "macro_nel": wl.nel, "rve_per_gpu": n_rve_run / world,
              "factorization": "tile-sparse" if args.tile_sparse else "dense", "macro_basis": args.macro_basis,
              "rve_ordering": args.rve_ordering, "macro_precond": args.macro_precond}

    if args.impl == "reference":
        if rank != 0:
            return
        times, cores = oracle_full_steps(wl, args.warmup + args.steps)
        timed = times[min(args.warmup, len(times) - 1):] if len(times) > 1 else times
        t = statistics.median(timed)
        val = wl.n_rve / t
        what = ("full steps: every RVE condensed (skyline Cholesky, unit-strain route), direct macro solve, "
                "recovery of every RVE" if wl.kind == "linear" else
                "full Newton iterations: every RVE condensed at the reference state, direct macro solve")
        sample = (f"{len(timed)} timed of {len(times)} run ({args.warmup} warm-up requested, {args.steps} timed "
                  f"requested; the arm stops after 150 s of oracle work) -- {what}")
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "tangents/s", "n_gpus": world,
                "device": "host CPU (the oracle on rank 0; other ranks idle)",
                "steps": len(timed), "steps_requested": args.steps, "warmup": len(times) - len(timed),
                "ms_per_step": t * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": val, "unit": "tangents/s", "cores": cores, "kind": "oracle",
                                 "sample": sample, "cpu": cpu_model()},
                "e2e": {"value": val, "unit": "tangents/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import numpy as np
    import torch
    dist_on = world > 1 or args.sharded  # the sharded path (one rank per GPU, NCCL)
    if dist_on:
        import socket

        import torch.distributed as dist
        torch.cuda.set_device(local)
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_2312_12771_b200.hom import Homogenizer

    if dist_on:
        from paper_2312_12771_b200.dist import ShardedHomogenizer
        sh = ShardedHomogenizer(wl, tile_sparse=args.tile_sparse, macro_basis=args.macro_basis,
                                rve_ordering=args.rve_ordering, macro_precond=args.macro_precond)
        h = sh.h
    else:
        sh = None
        h = Homogenizer.from_workload(wl, tile_sparse=args.tile_sparse, macro_basis=args.macro_basis,
                                      rve_ordering=args.rve_ordering, macro_precond=args.macro_precond)
    work = h.work
    config["l2"] = (f"no flush: each step writes and re-reads the K_ff tile pool ({h.sizes.rve_count * work.g_tiles * 32768 / 1e9:.2f} GB, "
                    f"{work.g_tiles} 64x64 tiles per RVE), larger than the 126 MB L2")
    dev = torch.cuda.current_device()
    B, m = h.n_rve, h.m
    C = h.empty(B, m, m)
    u = h.empty(h.n_dof)
    w = h.empty(B, h.n_pad)
    P_eff = h.empty(B, m) if h.finite else None
    P_avg = h.empty(B, m) if h.finite else None
    F = h.empty(B, m) if h.finite else None
    du = h.empty(h.n_dof) if h.finite else None
    cg_iters = []

    if h.finite and sh is None:  # a mid-load state: one converged load step first, then time Newton iterations
        u0, _ = h.newton(1, tol=1e-9)
        u.copy_(u0)
    elif h.finite:  # sharded: the first Newton iterations of load step 1 (same per-iteration work)
        u.zero_()
        sh.newton_iteration(u, F, C, P_eff, P_avg, du, scale=1.0 / wl.n_steps)

    def step():
        if sh is not None:
            if h.finite:
                _, _, info = sh.newton_iteration(u, F, C, P_eff, P_avg, du)
            else:
                _, _, _, info = sh.solve_linear(C, u, w)
            cg_iters.append(info.iterations)
            return
        if h.finite:
            h.macro_kinematics(u, F)
            h.condense(F, C, P_eff, P_avg)
            h.macro_residual_norm(P_avg)
            h.micro_residual_max()
            _, info = h.macro_solve(C, P_eff, scale=0.0, x=du)
            h.newton_update(u, du)
        else:
            h.condense(None, C)
            _, info = h.macro_solve(C, None, 1.0, u)
            h.recover(u, w)
        cg_iters.append(info.iterations)

    def barrier():
        if dist_on:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.2)
    h.profile(True)
    n0 = h.launch_count()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = h.launch_count() - n0
    ms = e0.elapsed_time(e1)
    prof = h.profile_read()
    h.profile(False)
    clocks = sampler.stop()
    if dist_on:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = B * args.steps / (ms * 1e-3)  # B = all RVEs of the (sharded) problem when world > 1

    # ---------------- end to end: host inputs (pinned) -> C-ABI -> host results, every step
    # the same rows the context was built from (Homogenizer.from_workload: one RVE per element with the
    # constant basis takes the rows of the element's first Gauss-point RVE)
    stride = wl.n_qp if args.macro_basis == "constant" else 1
    ph_rows = wl.phase[::stride] if wl.phase.shape[0] > 1 else wl.phase[0]
    mt_rows = wl.mat[::stride] if wl.mat.shape[0] > 1 else wl.mat[0]
    ph_host = torch.from_numpy(np.ascontiguousarray(ph_rows)).pin_memory()
    mt_host = torch.from_numpy(np.ascontiguousarray(mt_rows)).pin_memory()
    C_host = torch.empty((B, m, m), dtype=torch.float64).pin_memory()
    u_host = torch.empty(h.n_dof, dtype=torch.float64).pin_memory()
    w_host = torch.empty((B, h.n_pad), dtype=torch.float64).pin_memory()

    # results of step k land in device set k % 2 (linear: written there directly; finite strain: a
    # device snapshot of the state), and their D2H copies run on a side stream, overlapped with
    # the next step -- every copy is still inside the timed region (e1 waits for the last one)
    side = torch.cuda.Stream()
    sets = [(C, u, w), (torch.empty_like(C), torch.empty_like(u), torch.empty_like(w))]
    snap = [(torch.empty_like(C), torch.empty_like(u)) for _ in range(2)]
    freed = [None, None]  # side-stream event: set k's copies are done
    k_step = [0]

    def step_e2e():
        nonlocal C, u, w
        k = k_step[0] % 2
        k_step[0] += 1
        if freed[k] is not None:
            stream.wait_event(freed[k])
        h.set_phases(ph_host, mt_host)
        if h.finite:
            step()
            Cs, us = snap[k]
            Cs.copy_(C, non_blocking=True)
            us.copy_(u, non_blocking=True)
            ws = None
        else:
            C, u, w = sets[k]
            step()
            Cs, us, ws = C, u, w
        done = torch.cuda.Event()
        done.record(stream)
        side.wait_event(done)
        with torch.cuda.stream(side):
            C_host.copy_(Cs, non_blocking=True)
            u_host.copy_(us, non_blocking=True)
            if ws is not None:
                w_host.copy_(ws, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(side)
        freed[k] = ev

    for _ in range(args.warmup):
        step_e2e()
    torch.cuda.synchronize()
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step_e2e()
    stream.wait_stream(side)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = e0.elapsed_time(e1)
    if dist_on:
        t = torch.tensor([ms_e2e], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_e2e = float(t.item())
    h2d = ph_host.numel() * ph_host.element_size() + mt_host.numel() * mt_host.element_size()
    d2h = C_host.numel() * 8 + u_host.numel() * 8 + (0 if h.finite else w_host.numel() * 8)

    if rank != 0:
        if dist_on:
            torch.distributed.destroy_process_group()
        return

    cond_ms, cond_n = prof["condense"]
    per_launch = min(h.sizes.rve_chunk, B)
    flop_rve = work.flop_executed if args.tile_sparse else wl.flop_per_rve()
    n_local = h.sizes.rve_count  # RVEs this rank condenses per step (all chunks)
    achieved = flop_rve * n_local * args.steps / (cond_ms * 1e-3) / 1e12 if cond_ms > 0 else None
    peak, peak_src = fp64_peak()
    dgemm = dgemm_live_tflops()
    step_ms_total = sum(v[0] for v in prof.values())
    breakdown = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                     "share": (v[0] / step_ms_total if step_ms_total else None)} for k, v in prof.items()}
    asm_ms = prof["rve_assemble"][0] / max(prof["rve_assemble"][1], 1)
    tr = (load_json(os.path.join(ROOT, "profiles", "traffic.json")) or {}).get(
        f"cfg{args.config}_{'tilesparse' if args.tile_sparse else 'dense'}")
    traffic = tr["dram_bytes"] if tr and tr.get("rve_per_launch") == per_launch and world == 1 else None
    # K1 writes the structurally nonzero K_ff tiles + the K_fe / r_f block + <C> (+ <P>)
    asm_bytes_rve = work.a_tiles * 32768 + h.sizes.n_tiles * 64 * 8 * 8 + 2 * 64 * 8
    algo = (f"{flop_rve:.4g} executed DMMA flop/RVE for the tile structure ({work.g_tiles} tiles, {work.gemm_tiles} GEMM + "
            f"{work.syrk_tiles} SYRK + {work.trsm_tiles} TRSM tile products; dense count {wl.flop_per_rve():.4g})"
            if args.tile_sparse else
            f"{wl.flop_per_rve():.4g} flop/RVE (n_f^3/3 + 2 n_f^2 m + n_f m^2, n_f={wl.n_f})")

    line = {
        "metric": METRIC, "value": value, "unit": "tangents/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "roofline": {"bound": "tensor", "kernel": "k_condense (K2-K4 fused FP64 DMMA Cholesky + solves + Schur)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_source": peak_src,
                     "peak_dgemm_live": dgemm, "frac_dgemm_live": (achieved / dgemm) if achieved else None,
                     "peak_dgemm_live_source": "cuBLAS DGEMM 8192^3 (torch.matmul f64), best of 10, this GPU, this run",
                     "algorithmic": f"{algo} x {n_local} RVEs per step ({max(cond_n, 1) // args.steps} launch(es) of "
                                    f"<= {per_launch} RVEs)"},
        "fp64_tflops_condense": achieved,
        "macro_solve_ms": (prof["macro_assemble"][0] + prof["cg"][0]) / args.steps,
        "cg_iterations": statistics.median(cg_iters) if cg_iters else None,
        "assembly": {"kernel": "k_rve_assemble (K1)", "ms_per_launch": asm_ms,
                     "GBps": asm_bytes_rve * h.sizes.rve_count * args.steps / (prof["rve_assemble"][0] * 1e-3) / 1e9
                     if prof["rve_assemble"][0] > 0 else None,
                     "bytes": f"{asm_bytes_rve} B/RVE: {work.a_tiles} structurally nonzero 64x64 K_ff tiles + K_fe + <C>"},
        "breakdown": breakdown,
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": {"value": B * args.steps / (ms_e2e * 1e-3), "unit": "tangents/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "what": "hom_set_phases from pinned host + condense + macro solve + recovery + D2H of C_eff, u, w (copies of step k overlap step k+1 on a side stream; all inside the timed region)"},
    }
    if world == 1 and not args.tile_sparse and not h.finite and args.macro_basis == "dirac":
        line["tile_sparse"] = tile_sparse_line(wl, C, args.steps, args.warmup, args.rve_ordering)
    if world == 1 and not args.no_companions and args.config == 3 and not args.tile_sparse:
        h.close()  # free the K_ff pool (up to 96 GB) before the companion contexts
        torch.cuda.empty_cache()
        line["companions"] = {f"cfg{c}": companion_line(c, max(args.steps, 20), args.warmup) for c in (2, 5)}
    if world == 1 and args.spmv_nel > 0:
        if m == 3:
            C_tile = C
        else:  # 2-D scaled mesh: plane-strain isotropic tangent (E = 1, nu = 0.3)
            lam, mu = 0.3 / (1.3 * 0.4), 1.0 / 2.6
            C_tile = torch.tensor([[[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]]],
                                  dtype=torch.float64, device="cuda")
        line["spmv_scaled"] = spmv_scaled(C_tile, args.spmv_nel)
    if world == 1 and not args.no_cpu_baseline:
        st, detail = oracle_step_time(wl)
        line["cpu_baseline"] = {"value": wl.n_rve / st, "unit": "tangents/s", "cores": detail["cores"],
                                "kind": "oracle", "sample": detail["sample"], "cpu": cpu_model(),
                                "per_core_value": detail["per_core_tangents_s"],
                                "per_core_sample": detail["per_core_sample"]}
    print(json.dumps(line))
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
