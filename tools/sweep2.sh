timeout 600 python -m pytest tests/test_gpu_dmma.py -x -q 2>&1 | tail -5 > gpurun_out/dmma_tests.log
timeout 1200 python tools/sweep.py C2,C3a,C4,C5-adv-P2,C5-adv-P1,C5-hyp-P1,C5-hyp-P2,C5-hyp-P4,C3b dmma,dmma-R2,dmma-S1,dmma-R2-S1,dmma-R4,dmma-b128-R2,dmma-b128-S1,dmma-c16-R2-S1,dmma-b64-R2,dmma-b64-S1,dmma-b128-R2-S1 8 > gpurun_out/sweep3.jsonl 2>&1
