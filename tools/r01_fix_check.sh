python -m pytest tests/test_gpu_pipeline.py -q -x 2>&1 | tail -3
FEMGPU_TUNE_CACHE=0 python tools/dbg_fused.py > gpurun_out/dbg_fused.log 2>&1
bash tools/r01_prof4.sh > gpurun_out/prof4.log 2>&1
