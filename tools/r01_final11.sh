export FEMGPU_TUNE_CACHE=0
python tools/forms_table.py C3b,C5-adv-P3,C5-hyp-P1,C5-hyp-P2,C5-adv-P4,C4 > gpurun_out/forms_table16.jsonl 2>&1
python -m pytest tests/test_gpu_tune.py -x -q > gpurun_out/gpu_tests11.log 2>&1
