O=gpurun_out/r2ba
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py -q -x > $O/tests.log 2>&1
timeout 900 python tools/trace_pairs.py > $O/trace.log 2>&1
timeout 900 python tools/trace_pairs.py > $O/trace2.log 2>&1
