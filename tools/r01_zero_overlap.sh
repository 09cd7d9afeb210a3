export FEMGPU_TUNE_CACHE=0
python -m pytest tests/test_gpu_pipeline.py -x -q 2>&1 | tail -3
for z in 0 1; do
  FEMGPU_ZERO_OVERLAP=$z python tools/forms_table.py C3b,C4,C5-adv-P3,C5-adv-P4,C5-hyp-P1,C5-hyp-P2,C5-hyp-P3,C5-hyp-P4 > gpurun_out/zd_${z}.jsonl 2>&1
done
