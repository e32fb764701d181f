timeout 600 python -m pytest tests/test_gpu_backward.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
for mb in 1 4 5 6 8; do HHB_JIT_BWD_MINB=$mb timeout 120 python tools/time_bwd.py; done
K=10 timeout 120 python tools/time_bwd.py
K=4 timeout 120 python tools/time_bwd.py
HHB_JIT_NOMERGE=1 timeout 120 python tools/time_bwd.py
