"""A few actions of one operator of a fused pair, or of the fused operator (for ncu captures).

usage: python tools/fused_run.py laplace+mass-P2 A|B|fused [reps]
"""
import sys

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402

name, which = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a, b = fg.fused_pair(name)
p = {"A": a, "B": b}.get(which) or fg.fuse_problems([a, b])[0]
with fg.GpuInstance(p) as g:
    for _ in range(reps):
        g.action()
print("done", name, which)
