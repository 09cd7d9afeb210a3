"""Times the auto schedule (and alternatives) on several benchmark configs; prints one JSON per config."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi

names = sys.argv[1].split(",")
peak = None
for name in names:
    t = time.time()
    try:
        p = fg.config_problem(name)
        g = fg.GpuInstance(p)
        build = time.time() - t
        if peak is None:
            peak = fg.fp64_peak()[0]
        flops = fg.usable_flops(p.signature) * p.connectivity.cell_count
        res = {"config": name, "cells": p.connectivity.cell_count, "dofs": p.output_size, "build_s": round(build, 1)}
        for label, s in [("auto", None), ("scpt", fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC))]:
            try:
                step, kern, zero = g.profile(s, warmup=3, reps=20)
                res[label] = {"step_us": round(step * 1e6, 1), "kernel_us": round(kern * 1e6, 1),
                              "gdofs": round(p.output_size / step / 1e9, 2),
                              "fp64_frac_kernel": round(flops / kern / 1e12 / peak, 3)}
            except Exception as e:
                res[label] = "FAILED: " + str(e)[:200]
        g.close()
        print(json.dumps(res), flush=True)
    except Exception as e:
        print(json.dumps({"config": name, "error": str(e)[:300]}), flush=True)
