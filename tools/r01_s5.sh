timeout 1200 python tools/sweep.py C5-hyp-P2,C5-hyp-P4,C4,C3a,C5-adv-P2,C5-hyp-P1,C3b dmma,dmma-R2-b128,dmma-R2-b128-q8,dmma-b128-q8,dmma-R2-q8,dmma-b128,dmma-R2-b64 6 > gpurun_out/sweep5.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_dmma.py -x -q 2>&1 | tail -3 > gpurun_out/dmma_tests.log
