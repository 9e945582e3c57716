O=gpurun_out/r2ad
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_nbody.py -x -q -k "heat or instrument or host_pipeline or matrix" > $O/tests.log 2>&1
timeout 600 python tools/heat_pairs.py > $O/heat_pairs.log 2>&1
