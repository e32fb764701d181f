timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest14.log 2>&1; tail -2 gpurun_out/pytest14.log
timeout 120 python tools/time_bwd.py
timeout 300 python tools/prof_torch.py c3 2>/dev/null | head -6; timeout 300 python tools/prof_torch.py c4 2>/dev/null| head -6
