for sh in 0 1 2 3 4 5; do echo "shape=$sh"; LAMB_NB_SHAPE=$sh python tools/nb_sweep.py 131072 auto 2>&1; done
