timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_tune.py -x -q 2>&1 | tail -5 > gpurun_out/sched_tests.log
timeout 1200 python tools/sweep.py C5-adv-P2,C3a,C5-hyp-P1,C5-adv-P1,C2 auto,scpt,scpt-g2,scpt-g3,scpt-g4,scpt-g2-smem,scpt-g2-const,scpt-g2-b64 8 > gpurun_out/sweep_scptg.jsonl 2>&1
