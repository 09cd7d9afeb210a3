"""Runs a few actions of a config under a named schedule (for ncu captures)."""
import sys

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from tools.sweep import sched

SCHED = {
    "auto": None,
    "scpt-atomic": fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC),
    "tile-128": fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=128),
    "tile-384": fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=384),
    "tile-256": fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=256),
    "macro6": fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=6),
}
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
label = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = int(sys.argv[4]) if len(sys.argv) > 4 else None
p = fg.config_problem(cfg, n=n)
with fg.GpuInstance(p) as g:
    for _ in range(reps):
        g.action(SCHED[label] if label in SCHED else sched(label))
print("done", cfg, label, reps)
