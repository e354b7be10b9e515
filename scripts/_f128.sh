FSE_VERBOSE=1 timeout 120 python scripts/geom_rates.py 128 2>&1 | cut -c1-120
FSE_LIB_PATH=$PWD/paper_2204_14193_b200/_diag/cld.so timeout 300 python scripts/slot_phase.py 4 128 2>&1 | cut -c1-400
