timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.log
for cfg in C4 C5-hyp-P2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:femgpu_dmma -s 2 -c 1 -o gpurun_out/ncu2_dmma_$cfg -f python tools/run_action.py $cfg dmma-R2-b128 3 > gpurun_out/ncu2_$cfg.log 2>&1
done
timeout 900 python tools/sweep.py C4,C5-hyp-P2,C5-adv-P1 dmma-R2-b128,dmma-R2-b128-S1,dmma-b128 5 > gpurun_out/sweep4.jsonl 2>&1
FEMGPU_DEBUG_NO_TVEC=1 timeout 900 python tools/sweep.py C4,C5-hyp-P2 dmma-R2-b128,dmma-R2-b128-S1 5 >> gpurun_out/sweep4.jsonl 2>&1
