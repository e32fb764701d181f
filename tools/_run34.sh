timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -q -x 2>&1 | tail -2
timeout 60 python tools/time_gemm.py 2>&1 | head -3
timeout 300 python tools/prof_torch.py c3 2>/dev/null | head -9; timeout 300 python tools/prof_torch.py c4 2>/dev/null| head -8
