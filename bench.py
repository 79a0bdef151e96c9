#!/usr/bin/env python
"""bench.py — AS-PCG end-to-end solve time for the RaNN + overlapping-Schwarz pipeline on B200.

Workload: BASELINE.json configs[1] (C2: 2-D multiscale Poisson, 16x16 subdomains, m=300, 60x60
points per subdomain = 921,600 collocation rows, PCA σ/σmax > 1e-6, AS-preconditioned CG on the
normal equations to relative residual 1e-10, FP64). One step = one full pipeline solve
(runner.hpp:202-275: PCA -> assembly -> equilibration -> normal blocks + Schwarz -> PCG -> test
evaluation) of one seed.

  value   seconds per solve, inputs (collocation points, boxes, random bases) already resident
          in HBM; CUDA events on the library's stream; max over ranks.
  e2e     the same metric through the public C-ABI call rdd_run_single with host inputs: host
          geometry/bases, pinned H2D of points and bases, D2H of the evaluation, every step.
  roofline  the block-sparse normal operator Hᵀ(H·w) (the matvec of the metric), HBM-bound.
  cpu_baseline  the CPU oracle (oracle/, C++ restatement of the reference) on a bounded slice.

N>1 (torchrun): replicas — every rank solves its own seed (seed + rank) on its own GPU; the
path has no data exchange in this tier. --impl reference runs the CPU
oracle on rank 0 only.
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

METRIC = "AS-PCG end-to-end solve sec to rel-res 1e-10; matvec HBM GB/s vs peak"
FALLBACK_HBM_GBS = 6650.0
# iterations of the full C2 solve measured on the device (used only to extrapolate the CPU sample)
FULL_ITERATIONS = {"C2": 173, "C1": 24}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        return world, rank, local, dist
    return 1, 0, 0, None


def reduce_max(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ CPU oracle sample
def cpu_sample(cfg_name: str, cfg, threads: int):
    """Time the CPU oracle on a slice of the workload and extrapolate to the full config.

    The slice keeps d, m, P (points per subdomain per axis) and the operator with
    2^d subdomains (corner boxes: ~15% fewer rows than interior ones, so a slight underestimate). Setup phases (PCA, assembly, local eigensolves) scale with the subdomain
    count; the solve scales with subdomains x iterations (the full-size iteration count is the
    device-measured one)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    from paper_2412_19207_b200 import configs

    J = 1
    for a in range(cfg.d):
        J *= cfg.counts[a]
    per = cfg.colloc[0] // cfg.counts[0]
    sl = [2] * cfg.d if J > 2 ** cfg.d else list(cfg.counts)[:cfg.d]
    scfg = configs.scaled(cfg, sl, per)
    Js = 1
    for v in sl:
        Js *= v
    o = Oracle(threads=threads)
    t0 = time.perf_counter()
    s = o.run_single(scfg)
    wall = time.perf_counter() - t0
    f = J / Js
    iters_full = FULL_ITERATIONS.get(cfg_name, s["iterations"])
    per_iter = s["t_solve"] / max(1, s["iterations"])
    est = (s["t_assemble"] + s["t_precond"]) * f + per_iter * f * iters_full + s["t_evaluate"] * f
    import oracle as orc_mod
    cores = orc_mod.lib().orc_max_threads()
    return {
        "value": est, "unit": "s", "cores": cores, "kind": "port",
        "sample": (f"CPU oracle (C++ restatement of the reference, OpenMP at the reference's 5 sites, "
                   f"LAPACK single-threaded as Eigen) timed on a {'x'.join(map(str, sl))}-subdomain slice of "
                   f"{cfg_name} (same m={cfg.m}, {per} points/subdomain/axis, {s['iterations']} PCG iterations, "
                   f"{wall:.1f} s wall), extrapolated x{f:.0f} subdomains and to {iters_full} iterations"),
        "slice_summary": {k: s[k] for k in ("J", "DoF", "N", "iterations", "t_assemble", "t_precond", "t_solve")},
    }


def run_reference(args, cfg, world, rank, dist):
    if rank != 0:
        return 0
    from paper_2412_19207_b200 import configs  # noqa: F401
    threads = os.cpu_count() or 1
    vals, last = [], None
    for i in range(args.warmup + args.steps):
        r = cpu_sample(args.config, cfg, threads)
        if i >= args.warmup:
            vals.append(r["value"])
            last = r
    v = statistics.median(vals)
    line = {
        "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (formula-defined problem, SplitMix64 bases as the reference)", "impl": "reference",
        "config": {"workload": args.config, **cfg.as_dict()},
        "cpu_baseline": {k: last[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ device arm
def run_device(args, cfg, world, rank, local, dist):
    from paper_2412_19207_b200 import abi as A
    from paper_2412_19207_b200 import rdd

    cfg.seed = cfg.seed + rank
    s = rdd.Solver(local)
    # setup step (untimed): builds and uploads the instance
    first = s.run_single(cfg)
    # the sampler starts before the warm-up so its own start-up (driver queries) stays outside the
    # timed region; it keeps sampling through it
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(1.0)
    for _ in range(args.warmup):
        s.rerun_resident()
    barrier(dist)
    l0 = s.launch_count()
    s.L.rdd_event_record(s.h, 0)
    summ = None
    for _ in range(args.steps):
        summ = s.rerun_resident()
    s.L.rdd_event_record(s.h, 1)
    import ctypes as C
    ms = C.c_double()
    s.L.rdd_event_elapsed(s.h, 0, 1, C.byref(ms))
    launches = (s.launch_count() - l0) / args.steps
    clk = clocks.stop()
    t_step = ms.value / 1e3 / args.steps
    t_step_max = reduce_max(dist, t_step)

    # e2e: the public API with host inputs (host setup + pinned H2D + compute + D2H) each step
    barrier(dist)
    h0, d0 = C.c_int64(), C.c_int64()
    s.L.rdd_io_bytes(C.byref(h0), C.byref(d0))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_s = s.run_single(cfg)
    e2e = (time.perf_counter() - t0) / args.steps
    h1, d1 = C.c_int64(), C.c_int64()
    s.L.rdd_io_bytes(C.byref(h1), C.byref(d1))
    e2e_max = reduce_max(dist, e2e)

    # roofline: the normal operator (two passes over H) timed back-to-back with CUDA events on
    # the library stream, same resident system
    op_form = cfg.op_form if cfg.op_form in (A.OPERATOR_TWO_PASS, A.OPERATOR_FUSED) else A.OPERATOR_TWO_PASS
    op_ms, op_bytes = s.bench_operator(op_form, reps=30)
    peak, peak_kind = peaks()
    achieved = op_bytes / (op_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_matvec_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("bytes_per_call")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample(args.config, cfg, os.cpu_count() or 1)
        except Exception as e:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": "s", "cores": 0, "kind": "port", "sample": f"failed: {e}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": t_step_max, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step_max * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (formula-defined problem, SplitMix64 bases as the reference)",
            "config": {"workload": args.config, "l2": "working set (S 3.1 GB, H 0.6 GB) exceeds the 126 MB L2",
                       "parallelism": f"replicas x{world} (one seed per GPU)", **cfg.as_dict()},
            "solves_per_s": world / t_step_max,
            "phases_s": {k: summ[k] for k in ("t_pca", "t_assemble", "t_precond", "t_solve", "t_evaluate")},
            "iterations": summ["iterations"], "converged": summ["converged"], "DoF": summ["DoF"], "N": summ["N"],
            "e_l2": summ["e_l2"], "final_residual": summ["final_residual"],
            "e2e": {"value": e2e_max, "unit": "s", "h2d_bytes_per_step": (h1.value - h0.value) // args.steps,
                    "d2h_bytes_per_step": (d1.value - d0.value) // args.steps},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": ("normal operator Hᵀ(H·w), single pass: k_fused_normal + k_fused_reduce" if op_form == A.OPERATOR_FUSED else "normal operator Hᵀ(H·w): k_block_gemv + k_block_gemv_t (y = H·w formed in its staging) + k_chunk_sum"),
                         "bytes_per_call": op_bytes, "ms_per_call": op_ms,
                         "nominal_peak": 8000.0, "frac_nominal": achieved / 8000.0},
            "clocks": clk,
        }
        if cpu is not None:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    s.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rdd", choices=["rdd", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local, dist = dist_setup()
    from paper_2412_19207_b200 import configs
    cfg = configs.aspcg(args.config)  # the metric: AS-PCG on every config
    try:
        if args.impl == "reference":
            rc = run_reference(args, cfg, world, rank, dist)
        else:
            rc = run_device(args, cfg, world, rank, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
