for mb in 1 4 5 6 8; do HHB_JIT_BWD_MINB=$mb timeout 120 python tools/time_bwd.py; done
