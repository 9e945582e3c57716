O=gpurun_out/r2ab
mkdir -p $O
timeout 600 python tools/misc_pairs.py > $O/misc_pairs.log 2>&1
timeout 900 python -m pytest tests/test_gpu_copy.py -x -q -k "split or matrix" > $O/tests.log 2>&1
