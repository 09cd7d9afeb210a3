"""e2e step time: synchronous femgpu_action_host vs streaming femgpu_action_host_async (pinned buffers).

usage: python tools/e2e_stream.py C2 [steps]
"""
import ctypes as C
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from paper_2506_17471_b200._native import lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = fg.config_problem(cfg)
ptrs = []


def pinned_like(a):
    ptr = C.c_void_p()
    lib().femgpu_host_alloc(a.nbytes, C.byref(ptr))
    b = np.ctypeslib.as_array((C.c_double * a.size).from_address(ptr.value))
    b[:] = a
    ptrs.append(ptr)
    return b


with fg.GpuInstance(p) as g:
    g.action()
    xs = [pinned_like(x) for x in p.scalar_inputs]
    vs = [pinned_like(x) for x in p.vector_inputs]
    ys = [pinned_like(np.zeros(p.output_size)) for _ in range(2)]
    for _ in range(3):
        g.action_host(xs, vs, ys[0])
    t0 = time.perf_counter()
    for _ in range(steps):
        g.action_host(xs, vs, ys[0])
    t_sync = (time.perf_counter() - t0) / steps
    for k in range(4):
        g.action_host_async(xs, vs, ys[k & 1])
    g.action_host_wait()
    t0 = time.perf_counter()
    for k in range(steps):
        g.action_host_async(xs, vs, ys[k & 1])
    g.action_host_wait()
    t_async = (time.perf_counter() - t0) / steps
    print(json.dumps({"config": cfg, "sync_ms": round(t_sync * 1e3, 3), "stream_ms": round(t_async * 1e3, 3),
                      "sync_gdofs": round(p.output_size / t_sync / 1e9, 3),
                      "stream_gdofs": round(p.output_size / t_async / 1e9, 3)}))
for ptr in ptrs:
    lib().femgpu_host_free(ptr)
