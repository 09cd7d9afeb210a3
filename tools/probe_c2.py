"""Quick probe: time the C2 flagship (P2 Laplace 3D, N=107) under several schedules."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 107
name = sys.argv[2] if len(sys.argv) > 2 else "C2"
t = time.time()
p = fg.config_problem(name, n=n)
print("build %.1fs cells=%d dofs=%d" % (time.time() - t, p.connectivity.cell_count, p.output_size), flush=True)
g = fg.GpuInstance(p)
print("create %.1fs" % (time.time() - t), flush=True)
sig = p.signature
flops = fg.usable_flops(sig) * p.connectivity.cell_count
res = {}
for label, s in [("auto", None),
                 ("scpt-atomic", fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC)),
                 ("scpt-atomic-256", fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, block_cells=256)),
                 ("tile-128", fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=128)),
                 ("tile-256", fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=256)),
                 ("tile-384", fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=384)),
                 ("tile-512", fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=512)),
                 ("tile-384-smem", fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=384, basis=abi.BASIS_SMEM))]:
    try:
        t0 = time.time()
        sec = g.time(s)
        res[label] = dict(us=sec * 1e6, gdofs=p.output_size / sec / 1e9, tflops=flops / sec / 1e12)
        print(label, json.dumps(res[label]), "(%.1fs)" % (time.time() - t0), flush=True)
    except Exception as e:
        print(label, "FAILED", e, flush=True)
print(json.dumps(res))
