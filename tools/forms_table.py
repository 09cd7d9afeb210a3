"""The benchmark-forms table: automatic schedule per config, step split, and the
fraction of the form roofline t_roof = max(bytes_alg / BW_HBM, flops_alg / F_FP64), F_FP64 = max of the
live DFMA and DMMA peaks.  One JSON line per config.

usage: python tools/forms_table.py [C1,C1b,...]   (default: every config)
"""
import json
import os

import numpy as np
import sys
import time

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from bench import ClockSampler, algorithmic_bytes, load_peaks  # noqa: E402


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(fg.CONFIGS)
    pk = fg.fp64_peaks()
    hbm = load_peaks().get("hbm_gbs") or 6545.9
    print(json.dumps({"peaks": pk, "hbm_gbs": hbm}), flush=True)
    for name in names:
        t0 = time.time()
        try:
            p = fg.config_problem(name)
            cells = p.connectivity.cell_count
            flops = fg.usable_flops(p.signature) * cells
            byts = algorithmic_bytes(p)
            t_roof = max(flops / (pk["fp64"] * 1e12), byts / (hbm * 1e9))
            with fg.GpuInstance(p) as g:
                g.action()
                with ClockSampler() as clk:
                    step, kern, zero = g.profile(warmup=3, reps=max(20, int(0.5 / max(g.time(min_reps=3, min_seconds=0.0), 1e-6))))
                plan = g.describe()
                # the timed path (fused zeroing / slabs when the tuner chose them) against the plain
                # [memset y, one launch] path, and twice in a row (no stale rows)
                y1 = np.array(g.action())
                y2 = np.array(g.action())
                os.environ["FEMGPU_ZERO_OVERLAP"] = "0"
                y0 = np.array(g.action())
                del os.environ["FEMGPU_ZERO_OVERLAP"]
                check = {"repeat_rel_l2": float(np.linalg.norm(y2 - y1) / np.linalg.norm(y0)),
                         "vs_one_launch_rel_l2": float(np.linalg.norm(y1 - y0) / np.linalg.norm(y0))}
            print(json.dumps({"config": name, "cells": cells, "dofs": p.output_size, "step_us": round(step * 1e6, 1),
                              "kernel_us": round(kern * 1e6, 1), "zero_us": round(zero * 1e6, 1),
                              "t_roof_us": round(t_roof * 1e6, 1),
                              "bound": "fp64" if flops / (pk["fp64"] * 1e12) >= byts / (hbm * 1e9) else "hbm",
                              "frac_step": round(t_roof / step, 3), "gdofs": round(p.output_size / step / 1e9, 2),
                              "plan": plan, "check": check, "clocks": clk.summary(), "wall_s": round(time.time() - t0, 1)}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"config": name, "error": str(e)[:300]}), flush=True)


if __name__ == "__main__":
    main()
