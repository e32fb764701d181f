#!/bin/bash
# BPTT occupancy sweep at the config-3 shape (tools/time_bwd.py)
for m in "$@"; do echo "BWD2_MINB=$m $(HHB_JIT_BWD2_MINB=$m python tools/time_bwd.py 2>&1 | tail -1)"; done
