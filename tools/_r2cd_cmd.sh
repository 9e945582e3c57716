O=gpurun_out/r2cd
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_copy.py -q -x > $O/tests.log 2>&1
timeout 900 python tools/jit_modes.py > $O/modes.log 2>&1
