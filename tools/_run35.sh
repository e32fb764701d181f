timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -q -x 2>&1 | tail -2
timeout 300 python tools/prof_torch.py c3 2>/dev/null | head -7
