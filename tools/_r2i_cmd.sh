O=gpurun_out/r2i
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_codec.py -q > $O/codec.log 2>&1
timeout 600 python tools/nb_shard_time.py > $O/shard.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_scale.py -x -q -k "nbody or c4" > $O/nb_tests.log 2>&1
