set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/m_on.log 2>&1; tail -1 gpurun_out/m_on.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MERGED', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"
HHB_JIT_NOMERGE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/m_off.log 2>&1; tail -1 gpurun_out/m_off.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NOMERGE', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"
