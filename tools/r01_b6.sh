timeout 600 python -m pytest tests/test_gpu_schedules.py -x -q -k "macro_y" 2>&1 | tail -3 > gpurun_out/ys_tests.log
timeout 900 python tools/sweep.py C2 auto,macro6-ys,macro6-ys-b32,macro6-ys-b128,macro6-ys-r128,macro6-ys-r96 10 > gpurun_out/sweep_ys.jsonl 2>&1
timeout 1200 python tools/sweep.py C4,C5-hyp-P2,C3a,C5-hyp-P1 dmma-R2-b128,dmma-R2-b128-m5,dmma-R2-b128-m6,dmma-b128-m6,dmma-b128-m8,dmma-b128-q8-m2,dmma-b128-q8-m3 6 > gpurun_out/sweep_minb.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_c2_launches.csv python bench.py --steps 200 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_under_ncu.log 2>&1
