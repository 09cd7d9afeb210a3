python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
export FEMGPU_TUNE_CACHE=0
python tools/forms_table.py > gpurun_out/forms_table14.jsonl 2>&1
unset FEMGPU_TUNE_CACHE
python bench.py > gpurun_out/bench_final8.json 2> gpurun_out/bench_final8.err
