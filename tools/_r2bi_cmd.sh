O=gpurun_out/r2bi
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_scale.py tests/test_gpu_codec.py -q -x -k "nbody or c4 or exact or sqrt" > $O/tests.log 2>&1
timeout 600 python tools/nb_exact_sweep.py > $O/exact_sweep.log 2>&1
for sh in 0 1 2; do LAMB_NB_EXACT_SHAPE=$sh timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "c4" > $O/scale_shape$sh.log 2>&1; done
