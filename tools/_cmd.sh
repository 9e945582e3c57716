python bench_suite.py C6 > gpurun_out/c6.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/c6.json'))
for k,v in d['C6_other_compositions_2^26'].items(): print(k, round(v['GB/s']), round(v['frac'],3))"
