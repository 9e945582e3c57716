O=gpurun_out/r2cv
mkdir -p $O
timeout 600 python tools/jit_latency.py > $O/latency.log 2>&1
