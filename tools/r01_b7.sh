./build/devspec_bench > gpurun_out/r01_devspec.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_tune.py tests/test_gpu_schedules.py -x -q 2>&1 | tail -5 > gpurun_out/tune_tests.log
./tests/cpp/build/test_adapter > gpurun_out/adapter.log 2>&1; echo "adapter rc $?" >> gpurun_out/adapter.log
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r01_c2_launches.csv python bench.py --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_under_ncu.log 2>&1
timeout 1800 python tools/forms_table.py > gpurun_out/forms_table4.jsonl 2>&1
