"""Steady-state cost of the reference's per-call API NeuralModel.train_step(batch) on pinned host
batches (cfg2).  (A variant replaying the cached host-fed step graph per call measured slower,
262 vs 240 us/call: its two syncs and stream plumbing cost more than the eager launches.)"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2207_11620_b200 import fields
from paper_2207_11620_b200.model import build_model
from paper_2207_11620_b200.sampler import InCoreSampler, SampleBatch
m = build_model(bench.CFG2, dims=bench.DIMS, seed=0)
fld = fields.rasterize(bench.FIELD, bench.DIMS)
smp = InCoreSampler(fld, seed=1)
host = []
for _ in range(8):
    bt = smp.sample(m.batch_size)
    host.append(SampleBatch(bt.coords.cpu().pin_memory(), bt.targets.cpu().pin_memory(), trusted=True))
for k in range(5):
    m.train_step(host[k % 8])
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for k in range(N):
    m.train_step(host[k % 8])
dt = (time.perf_counter() - t0) / N
print("us/call", dt * 1e6, "samples/s", m.batch_size / dt)
