"""Per-iteration time of CG on the device: femgpu_cg (libfemgpu, fused update kernels) vs the torch
loop of krylov.cg over DeviceOperator, against the action's own pipelined step.

usage: python tools/cg_bench.py [n] [iters]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 107
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
p = fg.symmetric_problem("helmholtz", 3, 2, 4, n)
dev = torch.device("cuda", 0)
b = torch.from_numpy(np.random.default_rng(5).uniform(0.5, 1.5, p.output_size)).to(dev)
with fg.GpuInstance(p) as g:
    g.action()
    step = g.time_steps(50, pipelined=True) / 50
    fg.krylov.native_cg(g, b, rtol=0.0, maxiter=5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, it_n, _ = fg.krylov.native_cg(g, b, rtol=0.0, maxiter=iters, check_every=iters)
    t_native = (time.perf_counter() - t0) / it_n
    op = fg.DeviceOperator(g)
    fg.cg(op.apply, b, rtol=0.0, maxiter=5, check_every=5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, it_t, _ = fg.cg(op.apply, b, rtol=0.0, maxiter=iters, check_every=iters)
    torch.cuda.synchronize()
    t_torch = (time.perf_counter() - t0) / it_t
print(json.dumps({"dofs": int(p.output_size), "iters": iters, "action_step_us": round(step * 1e6, 1),
                  "native_cg_us_per_iter": round(t_native * 1e6, 1), "torch_cg_us_per_iter": round(t_torch * 1e6, 1)}))
