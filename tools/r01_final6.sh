python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
export FEMGPU_TUNE_CACHE=0
python tools/forms_table.py > gpurun_out/forms_table12.jsonl 2>&1
unset FEMGPU_TUNE_CACHE
python bench.py > gpurun_out/bench_final6.json 2> gpurun_out/bench_final6.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref6.json 2> gpurun_out/bench_ref6.err
