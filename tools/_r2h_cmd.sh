O=gpurun_out/r2h
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_codec.py -x -q > $O/codec.log 2>&1
timeout 900 python -m pytest tests/test_gpu_copy.py -x -q > $O/copy_tests.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k "c3" > $O/c3.log 2>&1
