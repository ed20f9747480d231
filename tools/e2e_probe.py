"""Host issue cost vs device time of the host-fed training pipeline (cfg2, pinned batches)."""
import os, sys, time, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2207_11620_b200 import fields
from paper_2207_11620_b200.model import build_model
from paper_2207_11620_b200.sampler import InCoreSampler, SampleBatch
from paper_2207_11620_b200.trainer import StepPipeline, train

m = build_model(bench.CFG2, dims=bench.DIMS, seed=0)
m.train_mode = 1
fld = fields.rasterize(bench.FIELD, bench.DIMS)
smp = InCoreSampler(fld, seed=1)
B = m.batch_size
host = []
for _ in range(16):
    bt = smp.sample(B)
    host.append(SampleBatch(bt.coords.cpu().pin_memory(), bt.targets.cpu().pin_memory(), trusted=True))

class HB:
    def __init__(self): self.i = 0
    def sample(self, b):
        self.i += 1
        return host[self.i % len(host)]

hs = HB()
pipe = StepPipeline(m, hs, capacity=2000)
pipe.step(4); torch.cuda.synchronize()
N = 300
t_issue = []
ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
w0 = time.perf_counter(); ev0.record()
for _ in range(N):
    a = time.perf_counter(); pipe.step(1); t_issue.append(time.perf_counter() - a)
ev1.record(); torch.cuda.synchronize(); w1 = time.perf_counter()
print(json.dumps({"issue_us_median": float(np.median(t_issue)) * 1e6, "issue_us_p90": float(np.percentile(t_issue, 90)) * 1e6,
                  "wall_us_per_step": (w1 - w0) / N * 1e6, "gpu_us_per_step": ev0.elapsed_time(ev1) / N * 1e3}))
# split the issue cost
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable()
for _ in range(200): pipe.step(1)
pr.disable(); torch.cuda.synchronize()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14); print(s.getvalue()[:3500])
# the public API, as bench.py's e2e measures it
for steps in (4, 50, 50, 200):
    torch.cuda.synchronize()
    a = time.perf_counter()
    h = train(m, hs, steps=steps)
    torch.cuda.synchronize()
    print("train() steps", steps, "us/step", (time.perf_counter() - a) / steps * 1e6, flush=True)
