export FEMGPU_TUNE_CACHE=0
python -m pytest tests/test_gpu_pipeline.py -x -q -k overlapped 2>&1 | grep -E "assert|Error|passed|failed" | head -20
python tools/forms_table.py > gpurun_out/fz2.jsonl 2>&1
