"""Duplex PCIe throughput of chunked copies (the e2e pipeline's pattern), pinned buffers, CUDA events.

usage: python tools/pcie_chunks.py [chunks] [ways]
  Each chunk is split over `ways` streams per direction.
  h2d / d2h: one direction alone; a: both directions, no dependencies;
  b: D2H chunk k waits for H2D chunk k (the pipeline's dependency, no kernel)
"""
import json
import sys

import torch

n = 9938375
K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
up = [torch.cuda.Stream() for _ in range(W)]
dn = [torch.cuda.Stream() for _ in range(W)]
cut = [n * k // K for k in range(K + 1)]


def run(mode):
    for k in range(K):
        a, b = cut[k], cut[k + 1]
        parts = [a + (b - a) * w // W for w in range(W + 1)]
        evs = []
        if mode != "d2h":
            for w in range(W):
                with torch.cuda.stream(up[w]):
                    d_in[parts[w]:parts[w + 1]].copy_(h_in[parts[w]:parts[w + 1]], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(up[w])
                    evs.append(e)
        if mode == "h2d":
            continue
        for w in range(W):
            if mode == "b":
                for e in evs:
                    dn[w].wait_event(e)
            with torch.cuda.stream(dn[w]):
                h_out[parts[w]:parts[w + 1]].copy_(d_out[parts[w]:parts[w + 1]], non_blocking=True)


def timed(mode, reps=10):
    run(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    t = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record(main)
        for s in up + dn:
            s.wait_event(e0)
        run(mode)
        for s in up + dn:
            main.wait_stream(s)
        e1.record(main)
        torch.cuda.synchronize()
        t += e0.elapsed_time(e1)
    return t / reps


res = {"chunks": K, "ways": W, "bytes_each": n * 8}
for m in ("h2d", "d2h", "a", "b"):
    res[m + "_ms"] = round(timed(m), 3)
print(json.dumps(res))
