timeout 600 python -m pytest tests/test_gpu_tune.py -x -q 2>&1 | tail -5 > gpurun_out/tune_tests.log
timeout 1500 python tools/forms_table.py > gpurun_out/forms_table.jsonl 2>&1
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
