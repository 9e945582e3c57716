O=gpurun_out/r2cf
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_scale.py -q -x -k "c5" > $O/scale_c5.log 2>&1
timeout 1500 python bench_suite.py C5 C6 > $O/suite_c5c6.json 2> $O/suite.err
