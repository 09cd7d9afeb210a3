timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_r01_ref.json 2> gpurun_out/bench_r01_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_c2_launches.csv python bench.py --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:femgpu_ -s 8 -c 1 -o gpurun_out/r01_c2_full -f python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full.log 2>&1
FEMGPU_TUNE_CACHE=0 timeout 2400 python tools/forms_table.py > gpurun_out/forms_table8.jsonl 2>&1
