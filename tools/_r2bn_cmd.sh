O=gpurun_out/r2bn
mkdir -p $O
for mb in 0 3 4 6; do echo "== minB $mb" >> $O/modes.log; LAMB_JIT_MINB=$mb timeout 900 python tools/jit_modes.py >> $O/modes.log 2>&1; done
