python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_final10.json 2> gpurun_out/bench_final10.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref10.json 2> gpurun_out/bench_ref10.err
