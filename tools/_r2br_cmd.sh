O=gpurun_out/r2br
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_vec_transpose -s 2 -c 1 -o $O/vt python tools/prof_copy.py --src aos-packed --dst soa-mb > $O/ncu_vt.log 2>&1
ncu -i $O/vt.ncu-rep --page raw --csv > $O/vt_raw.csv 2>/dev/null
ncu -i $O/vt.ncu-rep --page details --csv > $O/vt_details.csv 2>/dev/null
rm -f $O/vt.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 1 > $O/ncu_bench.log 2>&1
