"""CPU-side timeline of one pipelined simulate(numpy) call (which stage waits)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_21407_b200 import _pipeline, dynamics as Dy, defaults as DF

p = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
i = (2.0 * np.random.default_rng(0).poisson(2.0, size=(20, 10_000_000))).astype(np.float32)
orig_copy, orig_sync = _pipeline._par_copy, torch.cuda.Event.synchronize
T0 = [0.0]
log = []
def pc(dst, src):
    t = time.perf_counter(); orig_copy(dst, src); log.append(("host copy", t - T0[0], time.perf_counter() - t))
def es(self):
    t = time.perf_counter(); orig_sync(self); log.append(("event wait", t - T0[0], time.perf_counter() - t))
_pipeline._par_copy = pc
torch.cuda.Event.synchronize = es
for k in range(3):
    log.clear(); T0[0] = time.perf_counter()
    tr = Dy.simulate(p, i); torch.cuda.synchronize()
    tot = time.perf_counter() - T0[0]
    del tr
print("total %.1f ms" % (tot * 1e3))
for name, at, dur in log:
    print("%-11s at %7.1f ms  took %6.1f ms" % (name, at * 1e3, dur * 1e3))
for chunk in (64 << 20, 128 << 20, 512 << 20):
    _pipeline.CHUNK_BYTES = chunk
    for k in range(2):
        t = time.perf_counter(); tr = Dy.simulate(p, i); torch.cuda.synchronize(); el = time.perf_counter() - t; del tr
    print("chunk %4d MB: %.1f ms" % (chunk >> 20, el * 1e3))
