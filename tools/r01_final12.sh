python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
export FEMGPU_TUNE_CACHE=0
python tools/forms_table.py > gpurun_out/forms_table17.jsonl 2>&1
