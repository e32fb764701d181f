#!/bin/bash
# config-3 step timing under BPTT occupancy variants (tools/time_c3.py)
for m in "$@"; do HHB_JIT_BWD2_MINB=$m python tools/time_c3.py bf16 2>&1 | tail -1; done
