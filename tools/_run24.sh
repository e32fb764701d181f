timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest24.log 2>&1; tail -2 gpurun_out/pytest24.log
HHB_JIT_BWD_VEC1=1 timeout 120 python tools/time_bwd.py
for mb in 4 6 8 10; do HHB_JIT_BWD2_MINB=$mb timeout 120 python tools/time_bwd.py; done
