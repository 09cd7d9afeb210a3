import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import dist as fdist, abi
from oracle import oracle
p = fg.config_problem("C4", n=8)
print("full", np.linalg.norm(fg.gpu_action(p) - oracle.reference_action(p)) / np.linalg.norm(oracle.reference_action(p)))
for pl in fdist.plan(p, 2):
    loc = pl.local
    ref = oracle.reference_action(loc)
    for name, s in [("auto", None), ("scpt", fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC)), ("dmma", fg.TilingParams.dmma())]:
        with fg.GpuInstance(loc) as g:
            y = g.action(s)
            print(pl.rank, name, np.linalg.norm(y - ref) / np.linalg.norm(ref), g.describe(s)[:80])
