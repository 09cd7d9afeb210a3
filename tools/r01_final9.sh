python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_tune.py -x -q > gpurun_out/gpu_tests9.log 2>&1
export FEMGPU_TUNE_CACHE=0
python tools/forms_table.py C2,C3a,C4,C5-hyp-P1,C5-hyp-P2,C1b,C5-adv-P2 > gpurun_out/forms_table15.jsonl 2>&1
