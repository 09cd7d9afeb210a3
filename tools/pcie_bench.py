"""Host<->device copy ceilings for the e2e path: H2D alone, D2H alone, and both concurrently
(pinned host buffers, 80 MB each = the C2 x and y), CUDA events."""
import json
import torch

n = 9938375
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


res = {"bytes_each": n * 8, "h2d_ms": timed(h2d), "d2h_ms": timed(d2h), "both_ms": timed(both)}
res["h2d_gbs"] = n * 8 / res["h2d_ms"] / 1e6
res["d2h_gbs"] = n * 8 / res["d2h_ms"] / 1e6
res["both_gbs_total"] = 2 * n * 8 / res["both_ms"] / 1e6
print(json.dumps(res))
