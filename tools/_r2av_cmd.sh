O=gpurun_out/r2av
mkdir -p $O
timeout 1200 python tools/sweep_pairs.py > $O/sweep.log 2>&1
rm -f gpurun_out/jit_src.cu
