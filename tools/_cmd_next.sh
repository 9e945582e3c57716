python -m pytest tests/test_gpu_copy.py tests/test_gpu_codec.py -x -q 2>&1 | tail -3
python -c "
import sys; sys.path.insert(0,'.')
import torch, json
from paper_2302_08251_b200 import lamina as L
from bench_suite import run_suite
print(json.dumps(run_suite(L,0), indent=0)[:6000])
" 2>&1 | tail -120
python tools/nbody_prof.py && ncu --set full --clock-control none --import-source on -k regex:k_nbody -s 1 -c 1 -o gpurun_out/prof_nbody python tools/nbody_prof.py > gpurun_out/ncu_nb.log 2>&1; tail -2 gpurun_out/ncu_nb.log
