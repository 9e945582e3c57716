O=gpurun_out/r2j
mkdir -p $O
timeout 600 python tools/nb_shard_time.py > $O/shard.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_codec.py tests/test_gpu_copy.py -x -q > $O/tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_scale.py -x -q -k "nbody or c4" > $O/nb_tests.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
NCU="ncu --set full --clock-control none --import-source on -f"
timeout 600 $NCU -k regex:k_packv -c 1 -o $O/packv_u16 python tools/prof_copy.py --schema "Record{v:u16,w:u16}" --src soa-mb --dst bitpack-int:5 --reps 1 > $O/ncu1.log 2>&1
timeout 600 $NCU -k regex:k_pack32 -c 1 -o $O/pack32_e4m3 python tools/prof_copy.py --src soa-mb --dst bitpack-float:4,3 --reps 1 > $O/ncu2.log 2>&1
