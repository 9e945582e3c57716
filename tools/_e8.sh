timeout 200 python -c "
import json; from paper_2302_08251_b200 import lamina as L; from bench_suite import run_suite
r = run_suite(L, 0, parts=('C3',))['C3_bitpack_2^28']
print(json.dumps({k: r[k] for k in ('e5m10', 'e8m10', 'int12')}))" 2>&1 | tail -1
