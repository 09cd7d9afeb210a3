"""Debug: fused y zeroing vs one launch on C2-like instances (rel L2 between paths)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from tools.sweep import sched  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for n, nm in [(64, "macro6-qm-b32-m8"), (107, "macro6-qm-b32-m8"), (107, "macro6-b64"), (107, "scpt")]:
    p = fg.config_problem("C2", n=n)
    s = sched(nm)
    with fg.GpuInstance(p) as g:
        os.environ["FEMGPU_ZERO_OVERLAP"] = "0"
        ref = np.array(g.action(s))
        os.environ["FEMGPU_ZERO_OVERLAP"] = "1"
        out = []
        for i in range(3):
            y = np.array(g.action(s))
            out.append((g.stats()["launches_last_action"], rel(y, ref)))
        os.environ["FEMGPU_ZERO_OVERLAP"] = "0"
        y = np.array(g.action(s))
        out.append((g.stats()["launches_last_action"], rel(y, ref)))
        print(n, nm, out, flush=True)
del os.environ["FEMGPU_ZERO_OVERLAP"]
p = fg.config_problem("C2")
with fg.GpuInstance(p) as g:
    y = np.array(g.action())
    print("auto", g.describe().split(" | ")[0], g.stats()["launches_last_action"])
    y2 = np.array(g.action())
    os.environ["FEMGPU_ZERO_OVERLAP"] = "0"
    y3 = np.array(g.action())
    print("auto repeat", rel(y2, y), "vs one-launch", rel(y3, y), rel(y3, y2))
