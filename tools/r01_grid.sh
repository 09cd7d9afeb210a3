export FEMGPU_TUNE_CACHE=0
for gm in 1 2 4 0; do
FEMGPU_DMMA_GRID=$gm python tools/sweep.py C5-hyp-P1 dmma-c32-q4-b128-R1,dmma-c32-q4-b256-R1-S1 10 > gpurun_out/gr_hp1_$gm.jsonl 2>&1
FEMGPU_DMMA_GRID=$gm python tools/sweep.py C4,C5-hyp-P2,C5-hyp-P4,C5-adv-P3,C3b dmma-c32-q4-b128-R2,dmma-c32-q8-b128-R2,dmma-c32-q8-b128-R1,dmma-c32-q8-b256-R1-S1 10 > gpurun_out/gr_oth_$gm.jsonl 2>&1
done
python - <<'PY' > gpurun_out/occ.txt 2>&1
import paper_2506_17471_b200 as fg
from tools.sweep import sched
for cfg, nm in [("C5-hyp-P1","dmma-c32-q4-b128-R1"),("C4","dmma-c32-q4-b128-R2"),("C5-hyp-P2","dmma-c32-q8-b128-R2")]:
    p = fg.config_problem(cfg)
    with fg.GpuInstance(p) as g:
        g.action(sched(nm))
        print(cfg, nm, g.stats())
PY
