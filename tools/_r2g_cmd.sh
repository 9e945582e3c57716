O=gpurun_out/r2g
mkdir -p $O
timeout 600 python tools/nb_shard_time.py > $O/shard.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_scale.py -x -q -k "nbody or c4" > $O/nb_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_copy.py -x -q -k "bitpack or bool or criterion or float" > $O/copy_tests.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
