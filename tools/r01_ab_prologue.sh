# A/B: kernels with (repo) and without (wt_old, commit 126334c) the fused-zeroing prologue
export FEMGPU_TUNE_CACHE=0 FEMGPU_ZERO_OVERLAP=0
for rep in 1 2; do
for d in . wt_old; do
  (cd $d && python tools/sweep.py C5-adv-P2 scpt-b128-m5 20 > /root/repo/gpurun_out/ab_$(basename $d)_advp2_$rep.jsonl 2>&1)
  (cd $d && python tools/sweep.py C3a,C2,C5-adv-P1 scpt-g3-ql-b64,macro6-qm-b32-m8,macro6-b32-m8 20 > /root/repo/gpurun_out/ab_$(basename $d)_oth_$rep.jsonl 2>&1)
done; done
