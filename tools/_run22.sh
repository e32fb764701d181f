timeout 600 python -m pytest tests/test_gpu_learn.py tests/test_gpu_backward.py tests/test_gpu_layer.py -q 2>&1 | tail -2
timeout 300 python tools/prof_torch.py c3 2>/dev/null | head -12; timeout 300 python tools/prof_torch.py c4 2>/dev/null| head -3
