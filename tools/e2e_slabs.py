"""e2e (femgpu_action_host, pinned host buffers) per slab count of the overlapped pipeline.

usage: python tools/e2e_slabs.py C2 4,8,16,32,64 [steps] [edges]   (0 = the library default;
  edges: comma list of FEMGPU_PIPE_EDGE weights of the first and last slab, default 1)
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from paper_2506_17471_b200._native import lib  # noqa: E402

cfg = sys.argv[1]
slabs = [int(s) for s in sys.argv[2].split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
edges = [float(e) for e in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1.0]
p = fg.config_problem(cfg)
pinned = []


def pinned_like(a):
    ptr = C.c_void_p()
    lib().femgpu_host_alloc(a.nbytes, C.byref(ptr))
    buf = np.ctypeslib.as_array((C.c_double * a.size).from_address(ptr.value))
    buf[:] = a
    pinned.append(ptr)
    return buf


with fg.GpuInstance(p) as g:
    g.action()  # tune + JIT outside the timing
    xs = [pinned_like(x) for x in p.scalar_inputs]
    vs = [pinned_like(x) for x in p.vector_inputs]
    yh = pinned_like(np.zeros(p.output_size))
    for k in slabs:
        if k:
            os.environ["FEMGPU_PIPE_SLABS"] = str(k)
        else:
            os.environ.pop("FEMGPU_PIPE_SLABS", None)
        for e in edges:
            os.environ["FEMGPU_PIPE_EDGE"] = str(e)
            for _ in range(3):
                g.action_host(xs, vs, yh)
            t0 = time.perf_counter()
            for _ in range(steps):
                g.action_host(xs, vs, yh)
            t = (time.perf_counter() - t0) / steps
            print(json.dumps({"config": cfg, "slabs": k, "edge": e, "ms": round(t * 1e3, 3),
                              "gdofs": round(p.output_size / t / 1e9, 3)}), flush=True)
for ptr in pinned:
    lib().femgpu_host_free(ptr)
