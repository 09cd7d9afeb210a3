"""Diagnostics for the multi-rank bench path (two ranks may share one GPU with gloo)."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import torch, torch.distributed as dist
import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import dist as fdist
from paper_2506_17471_b200._native import lib
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
lib().femgpu_set_device(0)
cfg, n = sys.argv[1], int(sys.argv[2])
p = fg.config_problem(cfg, n=n)
pl = fdist.plan(p, world)[rank]
dev = torch.device("cuda", 0)
ys, yr, xs, xr = fdist._index_tensors(pl, dev)
g = fg.GpuInstance(pl.local)
y = torch.zeros(pl.local.output_size, dtype=torch.float64, device=dev)
g.action_device(y_dev=y.data_ptr(), stream=torch.cuda.current_stream(dev).cuda_stream or 1)
torch.cuda.synchronize()
y_local = y.cpu().numpy().copy()
loc_ref = g.action()
print(rank, "local action vs instance action", np.abs(y_local - loc_ref).max(), flush=True)
stream = torch.cuda.current_stream(dev)
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
fdist.exchange(pl, y, ys, yr, True, torch)
for _ in range(steps - 1):
    if pl.x_send or pl.x_recv:
        import ctypes as C
        xp = C.c_void_p()
        lib().femgpu_device_input(g.handle, 0, C.byref(xp))
        x = torch.as_tensor(fdist._CudaArray(xp.value, pl.local.scalar_inputs[0].size), device=dev)
        xs_, xr_ = fdist._index_tensors(pl, dev)[2:]
        fdist.exchange(pl, x, xs_, xr_, False, torch)
    g.action_device(y_dev=y.data_ptr(), stream=stream.cuda_stream or 1)
    fdist.exchange(pl, y, ys, yr, True, torch)
torch.cuda.synchronize()
with fg.GpuInstance(p) as gi:
    ref = gi.action()
own = pl.owned_mask
yo = y.cpu().numpy()[own]
print(rank, "owned rel err", np.linalg.norm(yo - ref[pl.test_global[own]]) / np.linalg.norm(ref[pl.test_global[own]]),
      "send", {q: len(v) for q, v in pl.y_send.items()}, "recv", {q: len(v) for q, v in pl.y_recv.items()}, flush=True)
dist.destroy_process_group()
