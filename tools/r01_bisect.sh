export FEMGPU_TUNE_CACHE=0
for rep in 1 2; do
for d in . wt_1812de2 wt_eea5638; do
  (cd $d && python tools/sweep.py C5-adv-P2 scpt-b128-m5,scpt 10 > /root/repo/gpurun_out/bis_$(basename $d)_$rep.jsonl 2>&1)
done; done
