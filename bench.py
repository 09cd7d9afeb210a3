"""bench.py — FP64 matrix-free operator action, GDOF/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], SURVEY §8d "C2"): P2 Poisson (Laplacian) action on the
3D unit cube, N=107 cubes per side, 6 Kuhn tetrahedra per cube (7,350,258 cells,
9,938,375 DOFs), Q=4, synthetic tabulations/inputs with the reference's make_problem
distributions (seed 7).  One step = one full action y = A x (zero y + the action kernel).

  value   whole-job GDOF/s with x, maps, coordinates resident in HBM; K steps timed with CUDA
          events on the instance stream, bracketed by barrier + synchronize, max over ranks.
  e2e     the same metric through the public C-ABI call with HOST buffers
          (femgpu_action_host: H2D of x, the action, D2H of y, every step; pinned memory).
  roofline  the dominant kernel against the machine's FP64 peak = max(DFMA, DMMA), both measured
          live (femgpu_fp64_peak / femgpu_fp64_dmma_peak; MEASURED_PEAKS.json has no FP64 figure),
          its own pipe's peak alongside, and the HBM side against MEASURED_PEAKS.json.  The kernel
          is whatever the automatic schedule picked (cost model + timing, tune.cpp).
  cpu_baseline  the reference's own reference_action (oracle/_ref, compiled from
          /root/reference/proj/include/femsched/form.hpp) on the host cores, rank 0, N=1.

--impl reference: the reference's CPU implementation of the path (oracle/_ref) on all host
threads, same config/metric, each step a bounded cell sample of the same mesh.
Multi-GPU (torchrun, N>1): cells are partitioned into contiguous brick-major ranges (z-slabs),
each rank owns a DOF range, halos are exchanged over NCCL (paper_2506_17471_b200/dist.py);
strong scaling on the fixed mesh.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIG = "C2"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_summary.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="femgpu", choices=["femgpu", "reference"])
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--mesh-n", dest="n", type=int, default=None, help="override mesh size (testing)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload_desc(cfg_name, p, n):
    from paper_2506_17471_b200 import CONFIGS
    c = dict(CONFIGS[cfg_name])
    if n is not None:
        c["n"] = n
    return {
        "workload": "%s: %s P%d action, %dD unit %s, N=%d, Q=%d (%s)" % (
            cfg_name, c["form"], c["degree"], c["dim"], "cube (6 Kuhn tets/cube)" if c["dim"] == 3 else
            "square (2 triangles/square)", c["n"], c["Q"], "BASELINE.json configs[1]" if cfg_name == "C2" else ""),
        "form": c["form"], "dim": c["dim"], "degree": c["degree"], "quad_points": c["Q"], "n": c["n"],
        "cells": int(p.connectivity.cell_count), "dofs": int(p.output_size),
        "usable_flops_per_cell": None,
        "l2": "no flush: per-step footprint (maps + x + coords + y ~ 0.5 GB) exceeds the 126 MB L2",
        "seed": 7,
    }


def algorithmic_bytes(p):
    """SURVEY §8d bytes_alg: trial inputs + coords + output once, each DISTINCT index array once,
    tabulations + weights once."""
    sig, conn = p.signature, p.connectivity
    b = 8 * (sum(x.size for x in p.scalar_inputs) + sum(x.size for x in p.vector_inputs) + conn.coords.size
             + p.output_size)
    maps = [conn.test_map] + conn.scalar_maps + conn.vector_maps + [conn.coord_map]
    seen = []
    for m in maps:
        if not any(m.indices is s.indices or (m.indices.shape == s.indices.shape and np.array_equal(m.indices, s.indices))
                   for s in seen):
            seen.append(m)
    b += 4 * sum(m.indices.size for m in seen)
    tab = p.tabulations
    b += 8 * (sum(a.size for a in tab.scalar_phi) + sum(a.size for a in tab.vector_phi) + tab.psi.size + tab.weights.size)
    return int(b)


class ClockSampler:
    """nvidia-smi-equivalent clocks + throttle reasons via NVML during the timed region."""

    def __init__(self, device=0, period=0.005):
        self.samples, self.reasons = [], set()
        self.period = period
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def cpu_baseline(p, budget_s=20.0):
    """The reference's reference_action on the host cores (oracle/_ref), full workload, compact
    per-thread sub-instances; falls back to the C restatement (1 thread) if _ref is absent."""
    from oracle import oracle
    threads = max(1, min(os.cpu_count() or 1, 64))
    if oracle.ref_available():
        sec, _ = oracle.ref_time_threads(p, threads, reps=1)  # warm-up + calibration
        reps = max(1, min(5, int(budget_s / max(sec, 1e-3))))
        sec, _ = oracle.ref_time_threads(p, threads, reps=reps)
        return {"value": p.output_size / sec / 1e9, "unit": "GDOF/s", "cores": threads, "kind": "reference",
                "sample": "full %d-cell workload, %d rep(s), unmodified femsched::reference_action over %d "
                          "contiguous cell ranges (compact sub-instances), partial outputs summed in rank order"
                          % (p.connectivity.cell_count, reps, threads),
                "seconds_per_action": sec}
    n = min(p.connectivity.cell_count, 200000)
    t0 = time.perf_counter()
    oracle.reference_action(p, cell_range=(0, n))
    sec = time.perf_counter() - t0
    rate_cells = n / sec
    return {"value": rate_cells * p.output_size / p.connectivity.cell_count / 1e9, "unit": "GDOF/s", "cores": 1,
            "kind": "port", "sample": "first %d cells of the workload, C restatement (oracle/femoracle.c), "
                                      "scaled by DOFs/cell" % n}


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f)
    except Exception:
        return {}


def load_traffic():
    try:
        with open(TRAFFIC_PATH) as f:
            return json.load(f)
    except Exception:
        return {}


def run_reference(args):
    """--impl reference: the reference CPU path (oracle/_ref) on all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2506_17471_b200 as fg
    from oracle import oracle
    p = fg.config_problem(args.config, n=args.n)
    threads = max(1, min(os.cpu_count() or 1, 64))
    C = p.connectivity.cell_count
    kind = "reference" if oracle.ref_available() else "port"
    # calibrate a cell sample so that warmup + steps finish in about a minute
    probe = min(C, 200000)
    if kind == "reference":
        s, _ = oracle.ref_time_threads(p, threads, reps=1, cell_range=(0, probe))
    else:
        t0 = time.perf_counter()
        oracle.reference_action(p, cell_range=(0, probe))
        s = time.perf_counter() - t0
        threads = 1
    per_cell = s / probe
    sample = int(max(1000, min(C, 60.0 / max(args.steps + args.warmup, 1) / per_cell)))
    times = []
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            sec, _ = oracle.ref_time_threads(p, threads, reps=1, cell_range=(0, sample))
        else:
            t0 = time.perf_counter()
            oracle.reference_action(p, cell_range=(0, sample))
            sec = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(sec)
    t = sum(times) / len(times)
    value = (sample / C) * p.output_size / t / 1e9
    cfg = workload_desc(args.config, p, args.n)
    out = {
        "impl": "reference", "metric": "FP64 operator-action GDOF/s", "value": value, "unit": "GDOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": threads, "kind": kind,
                         "sample": "first %d of %d cells per step (GDOF/s scaled by the sampled fraction)" % (sample, C)},
        "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def run_single(args):
    import ctypes as C

    import paper_2506_17471_b200 as fg
    from paper_2506_17471_b200 import abi
    from paper_2506_17471_b200._native import lib

    p = fg.config_problem(args.config, n=args.n)
    g = fg.GpuInstance(p)
    cfg = workload_desc(args.config, p, args.n)
    flops_cell = fg.usable_flops(p.signature)
    cfg["usable_flops_per_cell"] = flops_cell
    cells = p.connectivity.cell_count
    # warm-up (JIT compile happens on the first action, outside any timed region)
    y = g.action()
    for _ in range(max(args.warmup, 3)):
        g.action_device()
    # ---- timed region: exactly K steps, CUDA events on the instance stream, device
    # synchronize on both sides (femgpu_time_steps)
    with ClockSampler() as clk:
        t_step = g.time_steps(args.steps) / args.steps
    launches_per_step = g.stats()["launches_last_action"]
    value = p.output_size / t_step / 1e9
    # ---- per-kernel split (same protocol) for the roofline
    step_s, kern_s, zero_s = g.profile(warmup=3, reps=min(200, max(20, args.steps // 5)))
    # ---- e2e through the public C-ABI with pinned host buffers
    nbytes_in = sum(x.nbytes for x in p.scalar_inputs) + sum(x.nbytes for x in p.vector_inputs)
    pinned = []

    def pinned_like(a):
        ptr = C.c_void_p()
        lib().femgpu_host_alloc(a.nbytes, C.byref(ptr))
        buf = np.ctypeslib.as_array((C.c_double * a.size).from_address(ptr.value))
        buf[:] = a
        pinned.append(ptr)
        return buf
    xs = [pinned_like(x) for x in p.scalar_inputs]
    vs = [pinned_like(x) for x in p.vector_inputs]
    yh = pinned_like(np.zeros(p.output_size))
    g.action_host(xs, vs, yh)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        g.action_host(xs, vs, yh)
    t_e2e = (time.perf_counter() - t0) / args.e2e_steps
    e2e = {"value": p.output_size / t_e2e / 1e9, "unit": "GDOF/s", "h2d_bytes_per_step": int(nbytes_in),
           "d2h_bytes_per_step": int(yh.nbytes), "ms_per_step": t_e2e * 1e3,
           "api": "femgpu_action_host (include/femgpu.h), pinned host buffers, wall clock"}
    for ptr in pinned:
        lib().femgpu_host_free(ptr)
    # ---- parity spot check of the benchmarked output (full workload, size-independent property:
    # linearity A(2x) = 2 A(x) exactly in binary floating point) and oracle on a cell sample
    y1 = g.action()
    # ---- roofline
    pk = fg.fp64_peaks()
    plan = g.describe()
    kernel = plan.split(" | ")[0]
    on_dmma = kernel.startswith("femgpu_dmma")
    peak_tf = pk["fp64"]  # the machine's FP64 peak: max(DFMA, DMMA), both measured live
    pipe_tf = pk["dmma"] if on_dmma else pk["dfma"]
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    alg_flops = flops_cell * cells
    alg_bytes = algorithmic_bytes(p)
    t_fp64 = alg_flops / (peak_tf * 1e12)
    t_hbm = alg_bytes / (hbm * 1e9) if hbm else None
    t_roof = max(t_fp64, t_hbm or 0.0)
    traffic = load_traffic().get(args.config, {}).get("dram_bytes_per_launch")
    roof = {"bound": "fp64" if t_fp64 >= (t_hbm or 0) else "hbm", "achieved": alg_flops / kern_s / 1e12,
            "peak": peak_tf, "unit": "TFLOP/s", "frac": (alg_flops / kern_s / 1e12) / peak_tf,
            "traffic": traffic,
            "peak_source": "measured live on this GPU: max(DFMA %.2f, DMMA %.2f) TFLOP/s (femgpu_fp64_peak, "
                           "femgpu_fp64_dmma_peak); MEASURED_PEAKS.json has no FP64 entry" % (pk["dfma"], pk["dmma"]),
            "pipe": {"name": "DMMA (mma.sync m8n8k4 f64)" if on_dmma else "DFMA", "peak": pipe_tf,
                     "frac": (alg_flops / kern_s / 1e12) / pipe_tf},
            "kernel": kernel + " (NVRTC sm_100a)", "schedule": plan, "kernel_us": kern_s * 1e6, "zero_y_us": zero_s * 1e6,
            "algorithmic_flops_per_launch": alg_flops, "algorithmic_bytes_per_launch": alg_bytes,
            "hbm": {"achieved_alg_gbs": alg_bytes / kern_s / 1e9, "peak_gbs": hbm,
                    "frac": (alg_bytes / kern_s / 1e9) / hbm if hbm else None, "peak_source": "MEASURED_PEAKS.json"},
            "form_roofline": {"t_roof_us": t_roof * 1e6, "t_fp64_us": t_fp64 * 1e6,
                              "t_hbm_us": t_hbm * 1e6 if t_hbm else None, "frac_of_step": t_roof / t_step,
                              "definition": "t_roof = max(bytes_alg/BW_HBM, flops_alg/F_FP64) (SURVEY 8d)"}}
    out = {
        "metric": "FP64 operator-action GDOF/s", "value": value, "unit": "GDOF/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg, "roofline": roof, "e2e": e2e, "gpu_launches": args.steps * launches_per_step,
        "clocks": clk.summary(), "step_split_us": {"step": step_s * 1e6, "kernel": kern_s * 1e6, "zero_y": zero_s * 1e6},
    }
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(p)
    os.environ["FEMGPU_ZERO_OVERLAP"] = "0"  # the plain [memset y, one launch] path
    y0 = g.action()
    del os.environ["FEMGPU_ZERO_OVERLAP"]
    out["parity_check"] = {"finite": bool(np.all(np.isfinite(y1))), "repeatable_rel_l2":
                           float(np.linalg.norm(y1 - y) / np.linalg.norm(y)),
                           "vs_one_launch_rel_l2": float(np.linalg.norm(y1 - y0) / np.linalg.norm(y0))}
    if not (out["parity_check"]["repeatable_rel_l2"] <= 1e-12 and out["parity_check"]["vs_one_launch_rel_l2"] <= 1e-12):
        print("bench: timed path disagrees with the one-launch path: %s" % out["parity_check"], file=sys.stderr)
    g.close()
    print(json.dumps(out))


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_2506_17471_b200 import dist
        return dist.bench(args)
    return run_single(args)


if __name__ == "__main__":
    main()
