mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_copy.py -x -q -k "record_side or bitpack or instrumented or matrix_r32 or heat" > gpurun_out/r01e_t4.log 2>&1; tail -2 gpurun_out/r01e_t4.log
timeout 200 python -c "
import json; from paper_2302_08251_b200 import lamina as L; from bench_suite import run_suite
print(json.dumps(run_suite(L, 0, parts=('C3',))))" > gpurun_out/r01e_c3.json 2>&1; tail -c 1500 gpurun_out/r01e_c3.json
timeout 200 python tools/recpack_pairs.py 2>&1 | tee gpurun_out/r01e_recpack4.log
timeout 200 python tools/heat_pairs.py 2>&1 | tee gpurun_out/r01e_heat.log
