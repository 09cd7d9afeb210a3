"""Cell-partitioned action with ranks as threads sharing one GPU (csrc/halo.cu, in-process peer
pointers): per world size, the max-over-ranks step time of `femgpu_halo_time_steps` next to the
single-instance step, so the exchange overhead on one device is visible (on one GPU the ranks'
kernels share the SMs: the ideal step equals the single-instance step).

usage: python tools/halo_threads.py C2 [steps] [worlds]
"""
import json
import sys
import threading
import time

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from paper_2506_17471_b200 import dist as fdist  # noqa: E402
from tests.test_dist import ThreadGather  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
worlds = [int(w) for w in (sys.argv[3] if len(sys.argv) > 3 else "2,4").split(",")]

p = fg.config_problem(cfg)
with fg.GpuInstance(p) as g:
    g.action()
    g.time_steps(5)
    t1 = g.time_steps(steps) / steps
print(json.dumps({"config": cfg, "world": 1, "step_us": round(t1 * 1e6, 1), "mode": "single instance, [memset + action]"}),
      flush=True)
del p

for world in worlds:
    tg = ThreadGather(world)
    res = [None] * world

    def rank(r):
        from paper_2506_17471_b200._native import lib
        lib().femgpu_set_device(0)
        gather = tg.for_rank(r)
        t0 = time.perf_counter()
        plan = fdist.build_plan(fdist.config_slab(cfg, r, world), r, world, gather)
        di = fdist.DistInstance(plan, gather)
        t_setup = time.perf_counter() - t0
        for _ in range(5):
            di.action()
        di.check()
        gather(None)
        t = di.time_steps(steps) / steps
        di.check()
        res[r] = {"rank": r, "step_us": round(t * 1e6, 1), "cells": int(plan.local.connectivity.cell_count),
                  "boundary_cells": plan.boundary_cells, "halo_rows": plan.halo_rows(), "setup_s": round(t_setup, 1),
                  "schedule": di.inst.describe(di.params).split(" | auto: ")[0]}
        gather(None)
        di.close()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    print(json.dumps({"config": cfg, "world": world, "step_us": max(x["step_us"] for x in res),
                      "mode": "ranks as threads on one GPU, halo action (pull, boundary, push || interior, completion)",
                      "ranks": res}), flush=True)
