timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.log
timeout 1800 python tools/forms_table.py > gpurun_out/forms_table3.jsonl 2>&1
