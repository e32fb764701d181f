timeout 120 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -5
timeout 60 python tools/time_gemm.py
HHB_GEMM_NO2SM=1 timeout 60 python tools/time_gemm.py
