timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py tests/test_gpu_layer.py tests/test_gpu_network.py -q -x 2>&1 | tail -2
timeout 300 python tools/prof_torch.py c3 2>/dev/null | head -4; timeout 300 python tools/prof_torch.py c4 2>/dev/null| head -4
bash tools/bench_variants.sh "X=0"
