"""Offline (no GPU) SASS census of the emitted kernel per config: registers, spills and the
instruction mix per cell, against the form's usable FLOPs (FP64 floor vs issue floor).

usage: python tools/sass_mix.py C2,C4 [schedule]    (schedule names as in tools/sweep.py)
"""
import collections
import glob
import json
import os
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from tools.sweep import sched  # noqa: E402

SMALL_N = {2: 8, 3: 4}


def census(cubin, fun):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, cubin], capture_output=True, text=True).stdout
    ops = collections.Counter()
    for line in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            ops[m.group(2)] += 1
    res = subprocess.run(["cuobjdump", "-res-usage", cubin], capture_output=True, text=True).stdout
    regs = None
    lines = res.splitlines()
    for i, l in enumerate(lines):
        if re.search(r"Function %s:" % fun, l) and i + 1 < len(lines):
            m = re.search(r"REG:(\d+).*LOCAL:(\d+)", lines[i + 1])
            if m:
                regs = (int(m.group(1)), int(m.group(2)))
    return ops, regs


def main():
    cfgs = sys.argv[1].split(",")
    sname = sys.argv[2] if len(sys.argv) > 2 else "auto"
    for cfg in cfgs:
        c = fg.CONFIGS[cfg]
        p = fg.config_problem(cfg, n=SMALL_N[c["dim"]] * (2 if c["dim"] == 2 else 1))
        s = sched(sname)
        with tempfile.TemporaryDirectory() as d:
            os.environ["FEMGPU_CACHE"] = d
            src = fg.emit_source(p, s)
            fg.jit_check(p, s)
            cub = glob.glob(d + "/*.cubin")[0]
            fun = re.search(r'extern "C" __global__ void (?:__launch_bounds__\([^)]*\) )?(\w+)', src).group(1)
            ops, regs = census(cub, fun)
        G = 1
        m = re.search(r"grp \* (\d+) \+", src)
        if m:
            G = int(m.group(1))
        fp64 = sum(v for k, v in ops.items() if k in ("DFMA", "DMUL", "DADD", "DSETP", "DMMA"))
        total = sum(ops.values())
        uf = fg.usable_flops(p.signature)
        print(json.dumps({"config": cfg, "sched": sname, "kernel": fun, "regs_local": regs, "cells_per_thread": G,
                          "fp64_per_cell": round(fp64 / G, 1), "usable_dfma_per_cell": uf // 2,
                          "fp64_overhead": round(fp64 / G / (uf / 2), 3), "instr_per_cell": round(total / G, 1),
                          "issue_per_fp64": round(total / max(fp64, 1), 2),
                          "top": ops.most_common(10)}))


if __name__ == "__main__":
    main()
