O=gpurun_out/r2af
mkdir -p $O
rm -f gpurun_out/jit_src.cu
timeout 900 python tools/jit_pairs.py > $O/jit_pairs.log 2>&1
cp gpurun_out/jit_src.cu $O/ 2>/dev/null; head -c 200000 $O/jit_src.cu > $O/jit_src_head.cu; rm -f $O/jit_src.cu gpurun_out/jit_src.cu
