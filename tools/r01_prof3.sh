for spec in "C3a dmma-b128" "C5-hyp-P1 dmma-b256" "C5-adv-P2 dmma-b128-q8" "C5-adv-P1 dmma-R2-b128"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:femgpu_dmma -s 2 -c 1 -o gpurun_out/ncu3_$1 -f python tools/run_action.py $1 $2 3 > gpurun_out/ncu3_$1.log 2>&1
done
