O=gpurun_out/r2al
mkdir -p $O
timeout 900 python tools/jit_variants.py > $O/jit_variants.log 2>&1
