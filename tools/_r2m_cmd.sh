O=gpurun_out/r2m
mkdir -p $O
timeout 2400 python bench_suite.py > $O/suite.json 2> $O/suite.err
