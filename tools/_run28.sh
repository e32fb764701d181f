timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest28.log 2>&1; tail -2 gpurun_out/pytest28.log
bash tools/bench_variants.sh "X=0"
timeout 120 python tools/time_bwd.py
