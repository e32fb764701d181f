timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest9.log 2>&1; tail -3 gpurun_out/pytest9.log
for k in 1 10; do K=$k timeout 120 python tools/time_bwd.py; done
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench9.log 2>&1; tail -1 gpurun_out/bench9.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd', d['value'], 'fwd_bwd', d['fwd_bwd']['ms_per_step'], 'c4', d['c4_train_step']['ms_per_step'])"
STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/layer_launches3.csv python tools/prof_layer.py > gpurun_out/ncu9.log 2>&1; tail -1 gpurun_out/ncu9.log
