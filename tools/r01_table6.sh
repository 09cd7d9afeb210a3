FEMGPU_TUNE_CACHE=0 timeout 2400 python tools/forms_table.py > gpurun_out/forms_table6.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_tune.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/t6.log
