export FEMGPU_TUNE_CACHE=0
S=dmma-c32-q4-b128-R1,dmma-c32-q4-b256-R1-S1,dmma-c32-q4-b256-R1
FEMGPU_ZERO_OVERLAP=0 python tools/sweep.py C5-hyp-P1 $S 10 > gpurun_out/sl_hp1_off.jsonl 2>&1
for k in 2 4 8 16 32; do
FEMGPU_ZERO_OVERLAP=1 FEMGPU_ZERO_SLABS=$k python tools/sweep.py C5-hyp-P1 $S 10 > gpurun_out/sl_hp1_$k.jsonl 2>&1
done
S=dmma-c32-q8-b128-R1,dmma-c32-q8-b128-R2
FEMGPU_ZERO_OVERLAP=0 python tools/sweep.py C5-hyp-P4,C5-hyp-P2,C4 $S 10 > gpurun_out/sl_hp4_off.jsonl 2>&1
for k in 4 8 16; do
FEMGPU_ZERO_OVERLAP=1 FEMGPU_ZERO_SLABS=$k python tools/sweep.py C5-hyp-P4,C5-hyp-P2,C4 $S 10 > gpurun_out/sl_hp4_$k.jsonl 2>&1
done
