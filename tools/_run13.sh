timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest13.log 2>&1; tail -2 gpurun_out/pytest13.log
timeout 300 python tools/prof_torch.py c3 2>/dev/null | head -12
