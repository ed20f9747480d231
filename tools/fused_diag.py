"""Diagnostic timings of nvol_adam_encode_step (fused Adam + next encode) on the cfg2 model:
the fused kernel with a tiny encode batch (Adam sweep alone), with the full batch,
and the standalone Adam / encode kernels, across Adam-CTA fractions."""
import ctypes, json, os, subprocess, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_11620_b200 import _lib, fields
from paper_2207_11620_b200.model import build_model, MODE_TCGEN05, TRAIN_ENCODE_ONLY
from paper_2207_11620_b200.sampler import InCoreSampler
from paper_2207_11620_b200.trainer import StepPipeline
import bench

model = build_model(bench.CFG2, dims=bench.DIMS, seed=0)
model.train_mode = MODE_TCGEN05
fld = fields.rasterize(bench.FIELD, bench.DIMS)
pipe = StepPipeline(model, InCoreSampler(fld, seed=1), capacity=1000)
pipe.step(3)
torch.cuda.synchronize()
B = model.batch_size
stream = torch.cuda.current_stream()
cfg = model.encoder.config
off, res, ent, dense = model.encoder.c_tables()

def fused(b):
    ws = model._workspace(B)
    def fn(ev):
        ev[0].record(stream)
        _lib.call("nvol_adam_encode_step", _lib.ptr(model.flat_params), _lib.ptr(model.flat_grads),
                  _lib.ptr(model.flat_m), _lib.ptr(model.flat_v), model.flat_size, _lib.ptr(pipe.sched),
                  pipe.sched.numel() // 3, _lib.ptr(pipe.counter), *pipe.adam_consts, _lib.ptr(pipe.nan_state),
                  _lib.ptr(pipe.acc), None, pipe.t0, 0, 1.0 / B, _lib.ptr(pipe.work), _lib.ptr(pipe.bufs[1][0]), b,
                  off, res, ent, dense, cfg.n_levels, cfg.n_features_per_level, model.mlp.config.n_neurons,
                  model.mlp.config.n_hidden_layers, _lib.ptr(ws), ws.numel(), _lib.stream())
        ev[1].record(stream)
    return float(bench._event_ms(torch, fn)[0]) * 1e3

def enc():
    def fn(ev):
        ev[0].record(stream)
        c, t = pipe.bufs[1]
        model.fwd_bwd_device(c, t, pipe.acc, b_global=B, flags=TRAIN_ENCODE_ONLY)
        ev[1].record(stream)
    return float(bench._event_ms(torch, fn)[0]) * 1e3

def adam():
    def fn(ev):
        ev[0].record(stream)
        _lib.call("nvol_adam_train_step", _lib.ptr(model.flat_params), _lib.ptr(model.flat_grads),
                  _lib.ptr(model.flat_m), _lib.ptr(model.flat_v), model.flat_size, _lib.ptr(pipe.sched),
                  pipe.sched.numel() // 3, _lib.ptr(pipe.counter), *pipe.adam_consts, _lib.ptr(pipe.nan_state),
                  _lib.ptr(pipe.acc), None, pipe.t0, 0, 1.0 / B, _lib.ptr(pipe.ticket), _lib.stream())
        ev[1].record(stream)
    return float(bench._event_ms(torch, fn)[0]) * 1e3

out = {"adam_us": adam(), "encode_us": enc(), "frac": os.environ.get("NVOL_AE_ADAM_FRAC", "0.5"),
       "fused_b128_us": fused(128), "fused_full_us": fused(B)}
print(json.dumps(out), flush=True)
