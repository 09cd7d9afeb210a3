export FEMGPU_TUNE_CACHE=0
S=""
for m in 6 8 9 10 11 12 13 14 16; do S="$S,macro6-qm-b32-m$m"; done
for m in 3 4 5 6 7; do S="$S,macro6-qm-b64-m$m"; done
for m in 8 10 12 14; do S="$S,macro6-b32-m$m"; done
python tools/sweep.py C2 auto$S 30 > gpurun_out/c2_minblocks.jsonl 2>&1
S=""
for m in 6 8 10 12 14 16; do S="$S,macro6-qm-b32-m$m,macro6-b32-m$m"; done
python tools/sweep.py C5-adv-P1 auto$S 10 > gpurun_out/advp1_minblocks.jsonl 2>&1
