O=gpurun_out/r2r
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:k_heat_closed -c 1 -o $O/heat_closed python tools/prof_copy.py --src aos-packed --dst soa-mb --dst-wrap 2 --gran 64 --reps 1 > $O/ncu_heat.log 2>&1
