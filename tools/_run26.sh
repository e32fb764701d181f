timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_layer.py -q -x 2>&1 | tail -2
timeout 120 python tools/time_bwd.py; HHB_JIT_BWD_VEC1=1 timeout 120 python tools/time_bwd.py
