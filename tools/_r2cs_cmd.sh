O=gpurun_out/r2cs
mkdir -p $O
LAMB_JIT_LOG=1 timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_copy.py tests/test_gpu_guard.py -q -x > $O/tests.log 2>&1
timeout 1800 python tools/sweep_pairs.py > $O/sweep.log 2>&1
