O=gpurun_out/r2cb
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py -q -x -k "host_pipeline" > $O/tests.log 2>&1
