set -x
for cfg in C4 C5-hyp-P2; do
  ncu --set full --clock-control none --import-source on -k regex:femgpu_dmma -s 2 -c 1 -o gpurun_out/ncu_dmma_$cfg -f python tools/run_action.py $cfg dmma 3 > gpurun_out/ncu_$cfg.log 2>&1
done
python tools/sweep.py C2,C3a,C4,C5-adv-P2,C5-hyp-P1,C5-hyp-P2 dmma,dmma-b128 5 > gpurun_out/sweep_store.jsonl 2>&1 
FEMGPU_DEBUG_SCATTER_STORE=1 python tools/sweep.py C2,C3a,C4,C5-adv-P2,C5-hyp-P1,C5-hyp-P2 dmma,dmma-b128 5 >> gpurun_out/sweep_store.jsonl 2>&1
