O=gpurun_out/r2bu
mkdir -p $O
timeout 900 python tools/jit_modes.py > $O/modes.log 2>&1
LAMB_JIT_FENCE=1 timeout 900 python tools/jit_modes.py > $O/modes_fence.log 2>&1
