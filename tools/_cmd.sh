for c in 2 3 4 6 8 16; do echo "VEC_CTAS=$c"; LAMB_VEC_CTAS=$c python bench.py --warmup 3 --steps 5 --no-e2e --no-cpu > gpurun_out/b_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); p=d['per_pair_gbs']
print(round(d['value']), round(d['roofline']['achieved']), ' '.join(str(round(v)) for k,v in p.items()))"; done
