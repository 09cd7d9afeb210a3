export FEMGPU_TUNE_CACHE=0
python tools/forms_table.py C5-adv-P2 > gpurun_out/ap2_alone.jsonl 2>&1
python tools/forms_table.py C5-adv-P1,C5-adv-P2 > gpurun_out/ap2_after.jsonl 2>&1
python tools/forms_table.py C1,C5-adv-P2 > gpurun_out/ap2_after_c1.jsonl 2>&1
