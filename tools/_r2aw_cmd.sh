O=gpurun_out/r2aw
mkdir -p $O
timeout 900 python tools/trace_pairs.py > $O/trace.log 2>&1
