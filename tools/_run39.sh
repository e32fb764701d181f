timeout 600 python -c "
import sys, torch; sys.path.insert(0, '.')
import bench
dev = torch.device('cuda', 0)
r = bench.fwd_bwd_leg(torch, dev); print('c3', r['ms_per_step'], r['eager_ms_per_step'], r['cuda_graph'])
r = bench.c4_leg(torch, dev); print('c4', r['ms_per_step'], r['eager_ms_per_step'], r['cuda_graph'], r['loss'])
"
