O=gpurun_out/r2ap
mkdir -p $O
timeout 900 python tools/jit_uni.py > $O/jit_uni.log 2>&1
