timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest4.log 2>&1; tail -15 gpurun_out/pytest4.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench4.log 2>&1; tail -1 gpurun_out/bench4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd', d['value'], 'fwd_bwd', d['fwd_bwd']['ms_per_step'], 'c4', d['c4_train_step']['ms_per_step'])"
