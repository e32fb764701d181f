timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest30.log 2>&1; tail -2 gpurun_out/pytest30.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench30.log 2>&1; tail -1 gpurun_out/bench30.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('fwd', d['value'], d['roofline']['frac'], 'fwd_bwd', d['fwd_bwd']['ms_per_step'], 'c4', d['c4_train_step']['ms_per_step'], 'c5', d['c5_network']['ms_per_network_step'], 'morph', d['morphology']['value'], d['morphology']['ms_per_step'])"
