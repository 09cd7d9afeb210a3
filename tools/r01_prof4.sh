# C2 bench kernel after fused zeroing (8 slab launches per step): launch list + one full capture
python bench.py --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/prof4_bench.json 2> gpurun_out/prof4_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/c2_launches4.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/prof4_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:femgpu_macro -s 40 -c 1 -o gpurun_out/ncu4_c2 -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu4.log 2>&1
