timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest20.log 2>&1; tail -2 gpurun_out/pytest20.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench20.log 2>&1; tail -1 gpurun_out/bench20.log
