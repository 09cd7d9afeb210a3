export FEMGPU_TUNE_CACHE=0
python -m pytest tests/test_gpu_dmma.py -x -q 2>&1 | tail -3
for t in 1 0; do
  FEMGPU_DMMA_TICKETS=$t python tools/forms_table.py C3b,C4,C5-adv-P3,C5-adv-P4,C5-hyp-P1,C5-hyp-P2,C5-hyp-P3,C5-hyp-P4 > gpurun_out/tk_${t}.jsonl 2>&1
done
