python -m pytest tests/test_gpu_copy.py -q -x -k "pack or bit" 2>&1 | tail -1
for r in 1 2; do python bench_suite.py C3 2>&1 | python -c "
import json,sys; d=json.load(sys.stdin)
print(' '.join(f\"{k}:{v['pack_frac']:.3f}/{v['unpack_frac']:.3f}\" for k,v in d['C3_bitpack_2^28'].items()))"; done
