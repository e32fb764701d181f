timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q 2>&1 | tail -3
timeout 120 python tools/time_gemm.py
HHB_GEMM_NONPERSISTENT=1 timeout 120 python tools/time_gemm.py
