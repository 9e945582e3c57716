python -m pytest tests/test_gpu_copy.py -x -q 2>&1 | tail -3
python tools/sweep_env.py LAMB_VEC=1 LAMB_VEC=0,LAMB_UNI_WARP=0,LAMB_DIRECT=1 > gpurun_out/sweep9.log 2>&1
cat gpurun_out/sweep9.log
