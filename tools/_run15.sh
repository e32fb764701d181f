for e in "X=1" "HHB_JIT_NOMERGE=1" "HHB_NO_JIT=1"; do echo "== $e"; env $e timeout 300 python -m pytest tests/test_gpu_backward.py -x -q 2>&1 | tail -2; done
