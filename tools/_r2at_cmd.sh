O=gpurun_out/r2at
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_copy.py tests/test_gpu_guard.py -q -x > $O/tests.log 2>&1
timeout 900 python tools/jit_pairs.py > $O/jit_pairs.log 2>&1
rm -f gpurun_out/jit_src.cu
