"""Fused multi-operator action vs the separate actions (fuse.py): pipelined step times with the
automatic schedule (and named schedules), parity of the fused output against the separate outputs.

usage: python tools/fused_sweep.py stokes-P2,laplace+mass-P2 [n] [sched,...]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from tools.sweep import sched  # noqa: E402


def step(p, s=None, reps=30):
    with fg.GpuInstance(p) as g:
        y = g.action(s)
        g.time_steps(3, s, pipelined=True)
        t = g.time_steps(reps, s, pipelined=True) / reps
        return t, y, g.describe().split(" | auto: ")[0]


for name in sys.argv[1].split(","):
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
    names = sys.argv[3].split(",") if len(sys.argv) > 3 else ["auto"]
    a, b = fg.fused_pair(name, n=n)
    f, offs = fg.fuse_problems([a, b])
    for nm in names:
        s = sched(nm)
        ta, ya, pa = step(a, s)
        tb, yb, pb = step(b, s)
        tf, yf, pf = step(f, s)
        fa, fb = fg.split_output(yf, offs)
        rel = max(float(np.linalg.norm(fa - ya) / np.linalg.norm(ya)), float(np.linalg.norm(fb - yb) / np.linalg.norm(yb)))
        print(json.dumps({"pair": name, "sched": nm, "cells": int(a.connectivity.cell_count), "rows": offs,
                          "sep_us": [round(ta * 1e6, 1), round(tb * 1e6, 1)], "fused_us": round(tf * 1e6, 1),
                          "speedup": round((ta + tb) / tf, 3), "rel_l2_fused_vs_separate": rel,
                          "plans": [pa, pb, pf]}), flush=True)
