"""Distributed CG per iteration, ranks as threads on one GPU: femgpu_halo_cg (dots all-reduced GPU to
GPU) vs krylov.cg over DistOperator with host all-reduces (the thread gather).

usage: python tools/dist_cg_bench.py [world] [n] [iters]
"""
import json
import sys
import threading
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from paper_2506_17471_b200 import dist as fdist  # noqa: E402
from tests.test_dist import ThreadGather  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
args = ("helmholtz", 3, 2, 14, n)
tg = ThreadGather(world)
out = [None] * world


def rank(r):
    import torch
    from paper_2506_17471_b200._native import lib
    lib().femgpu_set_device(0)
    gather = tg.for_rank(r)
    slab = fdist.rank_slab(args, r, world)
    tab = slab.local.tabulations
    tab.psi = np.ascontiguousarray(np.transpose(tab.scalar_phi[0], (0, 2, 1)))
    plan = fdist.build_plan(slab, r, world, gather)
    di = fdist.DistInstance(plan, gather)
    try:
        with torch.cuda.stream(torch.cuda.ExternalStream(di.inst.stream())):
            b = torch.from_numpy((0.5 + 1e-3 * (plan.test_global % 89)) * plan.owned_mask).cuda()
            di.cg(b, rtol=0.0, maxiter=4, check_every=4)
            gather(None)
            t0 = time.perf_counter()
            _, it_n, _ = di.cg(b, rtol=0.0, maxiter=iters, check_every=iters)
            gather(None)
            t_native = (time.perf_counter() - t0) / it_n
            op = fg.krylov.DistOperator(di)
            owned = torch.from_numpy(plan.owned_mask.astype(np.float64)).cuda()

            def dot(a, c):
                return torch.tensor(sum(gather(float(torch.dot(a * owned, c)))), dtype=torch.float64, device=a.device)

            def apply(v, o):
                op.apply(v, o)
                o.mul_(owned)
            gather(None)
            t0 = time.perf_counter()
            _, it_t, _ = fg.krylov.cg(apply, b, rtol=0.0, maxiter=iters, check_every=iters, dot=dot)
            gather(None)
            t_torch = (time.perf_counter() - t0) / it_t
            out[r] = (t_native, t_torch, int(plan.local.output_size))
    finally:
        di.close()


th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
for t in th:
    t.start()
for t in th:
    t.join()
print(json.dumps({"world": world, "n": n, "iters": iters, "rows_per_rank": [o[2] for o in out],
                  "native_us_per_iter": round(max(o[0] for o in out) * 1e6, 1),
                  "host_allreduce_us_per_iter": round(max(o[1] for o in out) * 1e6, 1)}))
