O=gpurun_out/r2ce
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_guard.py -q -x > $O/tests.log 2>&1
timeout 900 python tools/planes_cmp.py > $O/planes.log 2>&1
