O=gpurun_out/r2ck
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_guard.py tests/test_gpu_jit.py -q -x -k "changetype or conversions or c5 or planes or bytesplit or matrix" > $O/tests.log 2>&1
timeout 900 python tools/planes_cmp.py > $O/planes.log 2>&1
LAMB_PLANES_PSTAGE=0 timeout 900 python tools/planes_cmp.py > $O/planes_off.log 2>&1
