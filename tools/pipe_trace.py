"""Timeline of one host-buffer action (femgpu_action_host) per slab: H2D chunk done, slab kernel done,
D2H chunk done (CUDA events, FEMGPU_PIPE_TRACE=1), with copies or kernels dropped for comparison.

usage: python tools/pipe_trace.py [config] [slabs]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from paper_2506_17471_b200._native import lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
p = fg.config_problem(cfg)
pinned = []


def pinned_like(a):
    ptr = C.c_void_p()
    lib().femgpu_host_alloc(a.nbytes, C.byref(ptr))
    b = np.ctypeslib.as_array((C.c_double * a.size).from_address(ptr.value))
    b[:] = a
    pinned.append(ptr)
    return b


with fg.GpuInstance(p) as g:
    g.action()
    xs = [pinned_like(x) for x in p.scalar_inputs]
    vs = [pinned_like(x) for x in p.vector_inputs]
    yh = pinned_like(np.zeros(p.output_size))
    if len(sys.argv) > 2:
        os.environ["FEMGPU_PIPE_SLABS"] = sys.argv[2]
    for skip in ["", "copies", "kernels"]:
        if skip:
            os.environ["FEMGPU_PIPE_TRACE_SKIP"] = skip
        for _ in range(3):
            g.action_host(xs, vs, yh)
        os.environ["FEMGPU_PIPE_TRACE"] = "1"
        print("# dropped:", skip or "nothing", flush=True)
        g.action_host(xs, vs, yh)
        os.environ.pop("FEMGPU_PIPE_TRACE")
for ptr in pinned:
    lib().femgpu_host_free(ptr)
