"""bench.py — FP64 matrix-free operator action, GDOF/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], SURVEY §8d "C2"): P2 Poisson (Laplacian) action on the
3D unit cube, N=107 cubes per side, 6 Kuhn tetrahedra per cube (7,350,258 cells,
9,938,375 DOFs), Q=4, synthetic tabulations/inputs with the reference's make_problem
distributions (seed 7).  One step = one full action y = A x: one full zeroing of an output
vector + the action kernel.  Steps go through femgpu_action_device_pipelined into two alternating
output buffers (the library zeroes the next step's output inside the action kernel, or with a
memset where that measures faster -- the automatic schedule decides per instance).

  value   whole-job GDOF/s with x, maps, coordinates resident in HBM; K steps timed with CUDA
          events on the instance stream, bracketed by barrier + synchronize, max over ranks.
  e2e     the same metric through the public C-ABI with HOST buffers: K streaming steps
          (femgpu_action_host_async + femgpu_action_host_wait), each uploading its x from pinned memory
          and downloading its y, step i+1's H2D overlapping step i's D2H; e2e.sync = one
          femgpu_action_host at a time.
  roofline  the step's kernel against the machine's FP64 peak = max(DFMA, DMMA), both measured
          live (femgpu_fp64_peak / femgpu_fp64_dmma_peak; MEASURED_PEAKS.json has no FP64 figure).
  cpu_baseline  the reference's own reference_action (oracle/_ref, compiled from
          /root/reference/proj/include/femsched/form.hpp) on the host cores, rank 0, N=1; its
          output is the parity check of the timed output (parity_vs_reference).
  forms   every benchmark configuration of SURVEY §8d (C1..C5) with the automatic schedule:
          step time, roofline fraction, parity against the reference CPU path.
  fused   operator pairs sharing their trial function (fuse.py): the fused action's step against
          the two separate actions' steps, parity of both parts against the reference.
  caller  femgpu_cg on C2's mesh (symmetric Helmholtz): time per CG iteration against the action's
          step, iterations to a 1e-10 relative residual.

--impl reference: the reference's CPU implementation of the path (oracle/_ref) on all host
threads, same config/metric, each step a bounded cell sample of the same mesh (built by
oracle/mesh_np.py: that process never loads libfemgpu).
Multi-GPU: `--gpus N` without torchrun launches N ranks itself (python -m torch.distributed.run);
under torchrun, cells are partitioned into contiguous brick-major ranges (z-slabs), each rank
builds only its slab, and halos move GPU to GPU inside libfemgpu (paper_2506_17471_b200/dist.py).
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
    ap.add_argument("--no-forms", dest="forms", action="store_false",
                    help="skip the table of every benchmark configuration (SURVEY 8d)")
    ap.add_argument("--forms-budget", type=float, default=900.0, help="seconds for the forms table")
    ap.add_argument("--ref-budget", type=float, default=20.0,
                    help="seconds of reference CPU work per forms row (full action if it fits, else complete rows)")
    ap.add_argument("--no-fused", dest="fused", action="store_false",
                    help="skip the fused multi-operator rows (fuse.py, PAPER.md:2477-2482)")
    ap.add_argument("--no-caller", dest="caller", action="store_false",
                    help="skip the caller row (femgpu_cg per iteration on C2's mesh)")
    return ap.parse_args()


def workload_desc(cfg_name, p, n):
    from paper_2506_17471_b200 import CONFIGS
    from paper_2506_17471_b200.form import usable_flops
    c = dict(CONFIGS[cfg_name])
    if n is not None:
        c["n"] = n
    return {
        "workload": "%s: %s P%d action, %dD unit %s, N=%d, Q=%d (%s)" % (
            cfg_name, c["form"], c["degree"], c["dim"], "cube (6 Kuhn tets/cube)" if c["dim"] == 3 else
            "square (2 triangles/square)", c["n"], c["Q"], "BASELINE.json configs[1]" if cfg_name == "C2" else ""),
        "form": c["form"], "dim": c["dim"], "degree": c["degree"], "quad_points": c["Q"], "n": c["n"],
        "cells": int(p.connectivity.cell_count), "dofs": int(p.output_size),
        "usable_flops_per_cell": int(usable_flops(p.signature)),
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def host_threads():
    return max(1, min(os.cpu_count() or 1, 64))


def parity(y, ref, rows=None):
    """rel L2 (north star, <= 1e-12) and the reference's elementwise relative error with its
    1e-30 guard (search.hpp:360-366, <= 1e-10), optionally on a subset of rows."""
    y = np.asarray(y)
    ref = np.asarray(ref)
    if rows is not None:
        y, ref = y[rows], ref[rows]
    rel_l2 = float(np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-300))
    max_rel = float(np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1e-30))) if ref.size else 0.0
    return {"rel_l2": rel_l2, "max_rel": max_rel, "rows_checked": int(ref.size),
            "pass": bool(rel_l2 <= 1e-12 and max_rel <= 1e-10 and np.all(np.isfinite(y)))}


def complete_rows(p, m):
    """Rows of y whose every contribution comes from cells [0, m): exactly the rows a
    reference run over that cell range must reproduce."""
    tm = p.connectivity.test_map.indices
    inside = np.zeros(p.output_size, dtype=bool)
    inside[tm[:m].ravel()] = True
    if m < tm.shape[0]:
        inside[tm[m:].ravel()] = False
    return np.nonzero(inside)[0]


def reference_check(p, y, budget_s=15.0, threads=None):
    """The reference's own reference_action (oracle/_ref, all host threads) against the GPU
    output y of the same instance: the full action when it fits the budget, else the complete
    rows of a contiguous cell sample sized to the budget.  Returns (parity, seconds, kind)."""
    from oracle import oracle
    threads = threads or host_threads()
    C = p.connectivity.cell_count
    if not oracle.ref_available():
        m = min(C, 20000)
        ref = oracle.reference_action(p, cell_range=(0, m))
        rows = complete_rows(p, m) if m < C else None
        return parity(y, ref, rows), None, "port (C restatement, %d cells)" % m
    probe = min(C, 20000)
    t_probe, _ = oracle.ref_time_threads(p, threads, reps=1, cell_range=(0, probe))
    est = t_probe * C / probe
    if est <= budget_s or probe == C:
        sec, ref = oracle.ref_time_threads(p, threads, reps=1)
        return parity(y, ref), sec, "full"
    m = int(max(probe, min(C, C * budget_s / est)))
    sec, ref = oracle.ref_time_threads(p, threads, reps=1, cell_range=(0, m))
    rows = complete_rows(p, m)
    return parity(y, ref, rows), sec, "complete rows of cells [0, %d) of %d (full reference ~%.0f s)" % (m, C, est)


def cpu_baseline(p, budget_s=20.0):
    """The reference's reference_action on the host cores (oracle/_ref), full workload, compact
    per-thread sub-instances; falls back to the C restatement (1 thread) if _ref is absent.
    Returns (cpu_baseline dict, reference output or None)."""
    from oracle import oracle
    threads = host_threads()
    if oracle.ref_available():
        sec, out = oracle.ref_time_threads(p, threads, reps=1)  # warm-up + calibration; kept for parity
        reps = max(1, min(5, int(budget_s / max(sec, 1e-3))))
        if reps > 1:
            sec, _ = oracle.ref_time_threads(p, threads, reps=reps)
        return {"value": p.output_size / sec / 1e9, "unit": "GDOF/s", "cores": threads, "kind": "reference",
                "cpu_model": cpu_model(), "logical_cpus": os.cpu_count(),
                "sample": "full %d-cell workload, %d rep(s), unmodified femsched::reference_action over %d "
                          "contiguous cell ranges (compact sub-instances), partial outputs summed in rank order"
                          % (p.connectivity.cell_count, reps, threads),
                "seconds_per_action": sec}, out
    n = min(p.connectivity.cell_count, 200000)
    t0 = time.perf_counter()
    oracle.reference_action(p, cell_range=(0, n))
    sec = time.perf_counter() - t0
    rate_cells = n / sec
    return {"value": rate_cells * p.output_size / p.connectivity.cell_count / 1e9, "unit": "GDOF/s", "cores": 1,
            "kind": "port", "cpu_model": cpu_model(), "logical_cpus": os.cpu_count(),
            "sample": "first %d cells of the workload, C restatement (oracle/femoracle.c), scaled by DOFs/cell" % n}, None


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
    """--impl reference: the reference CPU path (oracle/_ref) on all host threads.  The mesh comes
    from oracle/mesh_np.py, so this process loads only the reference's own code (no libfemgpu)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2506_17471_b200 as fg
    from oracle import mesh_np, oracle
    p = fg.config_problem(args.config, n=args.n, mesh_fn=mesh_np.mesh)
    threads = host_threads()
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
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                         "logical_cpus": os.cpu_count(),
                         "sample": "first %d of %d cells per step (GDOF/s scaled by the sampled fraction)" % (sample, C)},
        "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mesh": "oracle/mesh_np.py (numpy restatement of the structured mesh generator; no libfemgpu in this process)",
    }
    print(json.dumps(out))


def roofline_terms(p, peak_tf, hbm):
    from paper_2506_17471_b200.form import usable_flops
    flops = usable_flops(p.signature) * p.connectivity.cell_count
    bytes_ = algorithmic_bytes(p)
    t_fp64 = flops / (peak_tf * 1e12)
    t_hbm = bytes_ / (hbm * 1e9) if hbm else 0.0
    return flops, bytes_, t_fp64, t_hbm, max(t_fp64, t_hbm)


def form_row(name, pk, hbm, ref_budget):
    """One benchmark configuration with the automatic schedule: pipelined step time (the bench
    step), kernel-only time, roofline fraction, parity of the timed output against the reference."""
    import paper_2506_17471_b200 as fg
    t0 = time.perf_counter()
    p = fg.config_problem(name)
    with fg.GpuInstance(p) as g:
        g.action()  # JIT + automatic schedule
        step_s, kern_s, zero_s = g.profile(warmup=2, reps=10)
        # ~0.2 s timed, after ~0.1 s of warm-up steps (small configs: clocks up after the CPU-side checks)
        k = int(max(5, min(20000, 0.2 / max(step_s, 1e-6))))
        g.time_steps(int(max(3, min(10000, 0.1 / max(step_s, 1e-6)))), pipelined=True)
        with ClockSampler() as clk:
            t_step = g.time_steps(k, pipelined=True) / k
        launches = g.stats()["launches_last_action"]
        y = g.read_output()
        plan = g.describe()
    flops, bytes_, t_fp64, t_hbm, t_roof = roofline_terms(p, pk["fp64"], hbm)
    par, ref_s, ref_kind = reference_check(p, y, budget_s=ref_budget)
    return {"config": name, "cells": int(p.connectivity.cell_count), "dofs": int(p.output_size),
            "quad_points": int(p.signature.quad_points), "steps": k, "step_us": t_step * 1e6,
            "kernel_only_us": kern_s * 1e6, "memset_step_us": step_s * 1e6, "launches_per_step": launches,
            "t_roof_us": t_roof * 1e6, "bound": "fp64" if t_fp64 >= t_hbm else "hbm",
            "frac_step": t_roof / t_step, "gdofs": p.output_size / t_step / 1e9, "plan": plan.split(" | auto: ")[0],
            "parity_vs_reference": dict(par, reference=ref_kind, reference_seconds=ref_s),
            "clocks": clk.summary(), "wall_s": round(time.perf_counter() - t0, 1)}


def run_single(args):
    import ctypes as C

    import paper_2506_17471_b200 as fg
    from paper_2506_17471_b200._native import lib

    wall0 = time.perf_counter()
    p = fg.config_problem(args.config, n=args.n)
    g = fg.GpuInstance(p)
    cfg = workload_desc(args.config, p, args.n)
    cfg["l2"] = "no flush: per-step footprint (maps + x + coords + y ~ 0.5 GB) exceeds the 126 MB L2"
    # (what a step is lives outside `config`, which both arms share verbatim)
    step_definition = ("one full zeroing of an output vector + one full action; femgpu_action_device_pipelined "
                       "into two alternating outputs (next output zeroed inside the action kernel or by a memset, "
                       "as the automatic schedule measured faster)")
    flops_cell = cfg["usable_flops_per_cell"]
    cells = p.connectivity.cell_count
    # warm-up (JIT compile + automatic schedule on the first action, outside any timed region)
    y = g.action()
    g.time_steps(max(args.warmup, 3), pipelined=True)
    # ---- timed region: exactly K steps, CUDA events on the instance stream, device
    # synchronize on both sides (femgpu_time_steps_ex)
    with ClockSampler() as clk:
        t_step = g.time_steps(args.steps, pipelined=True) / args.steps
    launches_per_step = g.stats()["launches_last_action"]
    y_timed = g.read_output()  # the last timed step's output
    value = p.output_size / t_step / 1e9
    # ---- per-kernel split of the plain [memset y, action] step (same protocol), for reference
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
    yh2 = pinned_like(np.zeros(p.output_size))
    # one step at a time: femgpu_action_host (returns with y on the host)
    g.action_host(xs, vs, yh)
    # three trials of each mode, the median reported (host-side PCIe throughput varies run to run)
    sync_trials, e2e_trials = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            g.action_host(xs, vs, yh)
        sync_trials.append((time.perf_counter() - t0) / args.e2e_steps)
    t_sync = sorted(sync_trials)[1]
    # streaming steps: femgpu_action_host_async + one femgpu_action_host_wait; every step uploads its
    # inputs and downloads its y (alternating host outputs), step i+1's upload overlaps step i's download
    for k in range(4):
        g.action_host_async(xs, vs, (yh, yh2)[k & 1])
    g.action_host_wait()
    for _ in range(3):
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            g.action_host_async(xs, vs, (yh, yh2)[k & 1])
        g.action_host_wait()
        e2e_trials.append((time.perf_counter() - t0) / args.e2e_steps)
    t_e2e = sorted(e2e_trials)[1]
    y_last = (yh, yh2)[(args.e2e_steps - 1) & 1]
    e2e = {"value": p.output_size / t_e2e / 1e9, "unit": "GDOF/s", "h2d_bytes_per_step": int(nbytes_in),
           "d2h_bytes_per_step": int(yh.nbytes), "ms_per_step": t_e2e * 1e3,
           "api": "femgpu_action_host_async x K + femgpu_action_host_wait (include/femgpu.h): every step copies its "
                  "inputs from pinned host memory and its y back; step i+1's H2D overlaps step i's D2H; wall clock "
                  "from the first enqueue to the wait's return; median of 3 trials of K steps",
           "trials_ms": [round(t * 1e3, 4) for t in e2e_trials],
           "sync": {"value": p.output_size / t_sync / 1e9, "ms_per_step": t_sync * 1e3,
                    "api": "femgpu_action_host, one step at a time (returns with y on the host)",
                    "trials_ms": [round(t * 1e3, 4) for t in sync_trials]}}
    y_e2e = np.array(y_last)
    for ptr in pinned:
        lib().femgpu_host_free(ptr)
    # ---- roofline of the step's kernel (one launch per pipelined step: its duration is the step)
    pk = fg.fp64_peaks()
    plan = g.describe()
    kernel = plan.split(" | ")[0]
    on_dmma = kernel.startswith("femgpu_dmma")
    peak_tf = pk["fp64"]  # the machine's FP64 peak: max(DFMA, DMMA), both measured live
    pipe_tf = pk["dmma"] if on_dmma else pk["dfma"]
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    alg_flops, alg_bytes, t_fp64, t_hbm, t_roof = roofline_terms(p, peak_tf, hbm)
    kern_t = t_step / max(1, launches_per_step) if "pipe-memset" not in kernel else kern_s
    traffic = load_traffic().get(args.config, {}).get("dram_bytes_per_launch")
    roof = {"bound": "fp64" if t_fp64 >= t_hbm else "hbm", "achieved": alg_flops / kern_t / 1e12,
            "peak": peak_tf, "unit": "TFLOP/s", "frac": (alg_flops / kern_t / 1e12) / peak_tf,
            "traffic": traffic,
            "peak_source": "measured live on this GPU: max(DFMA %.2f, DMMA %.2f) TFLOP/s (femgpu_fp64_peak, "
                           "femgpu_fp64_dmma_peak); MEASURED_PEAKS.json has no FP64 entry" % (pk["dfma"], pk["dmma"]),
            "pipe": {"name": "DMMA (mma.sync m8n8k4 f64)" if on_dmma else "DFMA", "peak": pipe_tf,
                     "frac": (alg_flops / kern_t / 1e12) / pipe_tf},
            "kernel": kernel + " (NVRTC sm_100a)", "schedule": plan, "kernel_us": kern_t * 1e6,
            "kernel_duration": "CUDA events over the timed pipelined steps (%d launch(es)/step of this kernel, "
                               "in-kernel zeroing of the next output included)" % launches_per_step,
            "kernel_only_us_without_zeroing": kern_s * 1e6, "memset_zero_y_us": zero_s * 1e6,
            "algorithmic_flops_per_launch": alg_flops, "algorithmic_bytes_per_launch": alg_bytes,
            "hbm": {"achieved_alg_gbs": alg_bytes / kern_t / 1e9, "peak_gbs": hbm,
                    "frac": (alg_bytes / kern_t / 1e9) / hbm if hbm else None, "peak_source": "MEASURED_PEAKS.json"},
            "form_roofline": {"t_roof_us": t_roof * 1e6, "t_fp64_us": t_fp64 * 1e6,
                              "t_hbm_us": t_hbm * 1e6 if hbm else None, "frac_of_step": t_roof / t_step,
                              "definition": "t_roof = max(bytes_alg/BW_HBM, flops_alg/F_FP64) (SURVEY 8d)"}}
    out = {
        "metric": "FP64 operator-action GDOF/s", "value": value, "unit": "GDOF/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg, "step_definition": step_definition, "roofline": roof, "e2e": e2e,
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clk.summary(),
        "step_split_us": {"pipelined_step": t_step * 1e6, "memset_step": step_s * 1e6, "kernel_only": kern_s * 1e6,
                          "memset": zero_s * 1e6},
    }
    g.close()
    if not args.no_cpu_baseline:
        cb, ref = cpu_baseline(p)
        out["cpu_baseline"] = cb
        if ref is not None:
            out["parity_vs_reference"] = dict(parity(y_timed, ref), output="the last timed step's y",
                                              reference="oracle/_ref reference_action, full workload")
            out["parity_e2e_vs_reference"] = parity(y_e2e, ref)
    out["parity_check"] = {"finite": bool(np.all(np.isfinite(y_timed))),
                           "timed_vs_first_action_rel_l2": float(np.linalg.norm(y_timed - y) / np.linalg.norm(y))}
    del p, y, y_timed, y_e2e
    if args.forms:
        rows, skipped = [], []
        t_forms = time.perf_counter()
        for name in FORMS_ORDER:
            if name == args.config and args.n is None:
                continue
            if time.perf_counter() - t_forms > args.forms_budget:
                skipped.append(name)
                continue
            try:
                rows.append(form_row(name, pk, hbm, args.ref_budget))
            except Exception as e:  # noqa: BLE001 -- one failing config must not hide the others
                rows.append({"config": name, "error": str(e)[:300]})
        if args.n is None:
            c2 = {"config": args.config, "cells": cells, "dofs": int(cfg["dofs"]), "step_us": t_step * 1e6,
                  "kernel_only_us": kern_s * 1e6, "t_roof_us": t_roof * 1e6, "frac_step": t_roof / t_step,
                  "gdofs": value, "plan": plan.split(" | auto: ")[0], "parity_vs_reference": out.get("parity_vs_reference"),
                  "clocks": out["clocks"], "note": "the headline line above"}
            rows.insert(FORMS_ORDER.index(args.config), c2)
        ok = [r for r in rows if "frac_step" in r]
        out["forms"] = {"rows": rows, "skipped_for_time": skipped,
                        "at_least_half_roofline": sum(1 for r in ok if r["frac_step"] >= 0.5), "measured": len(ok),
                        "parity_pass": sum(1 for r in ok if (r.get("parity_vs_reference") or {}).get("pass")),
                        "definition": "frac_step = t_roof / pipelined step time (SURVEY 8d); automatic schedule; "
                                      "parity of the last timed step's y against the reference's reference_action"}
    if args.fused and args.n is None:
        out["fused"] = []
        for name in FUSED_ORDER:
            try:
                out["fused"].append(fused_row(name, args.ref_budget))
            except Exception as e:  # noqa: BLE001
                out["fused"].append({"pair": name, "error": str(e)[:300]})
    if args.caller and args.n is None:
        try:
            out["caller"] = caller_row()
        except Exception as e:  # noqa: BLE001
            out["caller"] = {"error": str(e)[:300]}
    out["wall_s"] = round(time.perf_counter() - wall0, 1)
    print(json.dumps(out))


def caller_row(iters=100):
    """The action's caller: femgpu_cg on C2's mesh with a symmetric Helmholtz operator,
    time per CG iteration against the action's own pipelined step, and the relative residual reached."""
    import torch

    import paper_2506_17471_b200 as fg
    from paper_2506_17471_b200.mesh import CONFIGS
    c = CONFIGS["C2"]
    p = fg.symmetric_problem("helmholtz", c["dim"], c["degree"], c["Q"], c["n"])
    b = torch.from_numpy(np.random.default_rng(5).uniform(0.5, 1.5, p.output_size)).cuda()
    with fg.GpuInstance(p) as g:
        g.action()
        step = g.time_steps(20, pipelined=True) / 20
        fg.krylov.native_cg(g, b, rtol=0.0, maxiter=4, check_every=4)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, it, _ = fg.krylov.native_cg(g, b, rtol=0.0, maxiter=iters, check_every=iters)
        t_it = (time.perf_counter() - t0) / it
        _, it_conv, rel = fg.krylov.native_cg(g, b, rtol=1e-10, maxiter=2000, check_every=10)
    return {"api": "femgpu_cg (csrc/cg.cu)", "problem": "C2 mesh, P2 Helmholtz with Psi = Phi^T (symmetric)",
            "dofs": int(p.output_size), "us_per_iteration": t_it * 1e6, "action_step_us": step * 1e6,
            "iterations_to_1e-10": it_conv, "rel_residual": rel}


FUSED_ORDER = ["laplace+mass-P2", "stokes-P2"]


def fused_row(name, ref_budget):
    """One fused pair: pipelined steps of A, of B and of the fused action (automatic schedules),
    parity of both parts of the fused output against the reference's reference_action."""
    import paper_2506_17471_b200 as fg
    t0 = time.perf_counter()
    a, b = fg.fused_pair(name)
    f, offs = fg.fuse_problems([a, b])

    def step(p):
        with fg.GpuInstance(p) as g:
            g.action()
            g.time_steps(3, pipelined=True)
            k = int(max(10, min(300, 0.2 / max(g.time_steps(1, pipelined=True), 1e-6))))
            t = g.time_steps(k, pipelined=True) / k
            return t, g.read_output(), g.describe().split(" | auto: ")[0]
    ta, _, pa = step(a)
    tb, _, pb = step(b)
    tf, yf, pf = step(f)
    parts = fg.split_output(yf, offs)
    checks = []
    for y, p in zip(parts, (a, b)):
        par, sec, kind = reference_check(p, y, budget_s=ref_budget)
        checks.append(dict(par, reference=kind))
    return {"pair": name, "cells": int(a.connectivity.cell_count), "rows": offs,
            "separate_step_us": [ta * 1e6, tb * 1e6], "fused_step_us": tf * 1e6, "speedup": (ta + tb) / tf,
            "plans": {"A": pa, "B": pb, "fused": pf}, "parity_vs_reference": checks,
            "pass": all(c["pass"] for c in checks), "wall_s": round(time.perf_counter() - t0, 1)}


FORMS_ORDER = ["C1", "C1b", "C2", "C3a", "C3b", "C4", "C5-adv-P1", "C5-adv-P2", "C5-adv-P3", "C5-adv-P4",
               "C5-hyp-P1", "C5-hyp-P2", "C5-hyp-P3", "C5-hyp-P4"]


def launch_ranks(args):
    """`--gpus N` without a launcher: start the N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and relay rank 0's JSON line."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.impl == "reference":
        return run_reference(args)
    if world > 1:
        from paper_2506_17471_b200 import dist
        return dist.bench(args)
    return run_single(args)


if __name__ == "__main__":
    main()
