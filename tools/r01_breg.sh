timeout 900 python -m pytest tests/test_gpu_dmma.py -x -q 2>&1 | tail -3 > gpurun_out/dmma_tests.log
timeout 1500 python tools/sweep.py C3a,C5-adv-P1,C5-hyp-P1,C2,C5-adv-P2,C4,C3b dmma-b128,dmma-breg-b128,dmma-breg-b256,dmma-breg-R2-b128,dmma-breg-q16-b128,dmma-breg-q12-b128 6 > gpurun_out/sweep_breg.jsonl 2>&1
