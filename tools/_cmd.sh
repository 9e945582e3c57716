python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for kb in 4 9; do echo KB=$kb; LAMB_WARP_TILE_KB=$kb python tools/misc_pairs.py 2>&1 | tail -12 | head -5; done
