"""Can the step's scatter (L2-RED bound) and Adam (HBM bound) overlap?  cfg2 tables, B = 65,536:
scatter alone, Adam alone, the two back to back on one stream, and the two launched on two
streams at once (Adam reads the scatter's gradient buffer, as in the step).  Timing only; the
concurrent launch races by construction."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2207_11620_b200 import _lib  # noqa: E402
from paper_2207_11620_b200.model import NAN_NONE, build_model  # noqa: E402

m = build_model(bench.CFG2, dims=bench.DIMS, seed=0)
b = 65536
cfg = m.encoder.config
nf = cfg.n_levels * cfg.n_features_per_level
c = torch.rand(b, 3, device="cuda")
dfm = torch.randn(nf, b, device="cuda") * 1e-3
off, res, ent, dense = m.encoder.c_tables()
n = m.flat_size
P, M, V = m.flat_params, m.flat_m, m.flat_v  # the model's own buffers (shared 128-byte alignment)
sched = torch.tensor([0.005, 0.1, 0.001], dtype=torch.float32, device="cuda")
counter = torch.zeros(1, dtype=torch.int64, device="cuda")
ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
acc = torch.zeros(1, dtype=torch.float64, device="cuda")
losses = torch.zeros(4, dtype=torch.float64, device="cuda")
ns = torch.tensor([NAN_NONE, 0], dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def scatter(s, lv=None):
    _lib.call("nvol_train_tc_scatter", _lib.ptr(c), _lib.ptr(dfm), b, b, off, res, ent, dense, cfg.n_levels,
              cfg.n_features_per_level, _lib.ptr(m.flat_grads), s.cuda_stream)


def adam(s, lo=0, hi=None):
    hi = n if hi is None else hi
    _lib.call("nvol_adam_train_step", _lib.ptr(P) + 4 * lo, _lib.ptr(m.flat_grads) + 4 * lo, _lib.ptr(M) + 4 * lo,
              _lib.ptr(V) + 4 * lo, hi - lo, _lib.ptr(sched), 1, _lib.ptr(counter), 0.9, 0.1, 0.999, 0.001, 1e-15,
              1e-6, _lib.ptr(ns), _lib.ptr(acc), _lib.ptr(losses), 0, 4, 1.0, _lib.ptr(ticket), s.cuda_stream)


main = torch.cuda.current_stream()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=30):
    ts = []
    for _ in range(reps):
        flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        fn()
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def both():
    ev = torch.cuda.Event()
    ev.record(main)
    sa.wait_event(ev)
    sb.wait_event(ev)
    scatter(sa)
    adam(sb)
    ja, jb = torch.cuda.Event(), torch.cuda.Event()
    ja.record(sa)
    jb.record(sb)
    main.wait_event(ja)
    main.wait_event(jb)


def serial():
    scatter(main)
    adam(main)


for _ in range(3):
    serial()
    both()
r = {"scatter": timed(lambda: scatter(main)), "adam": timed(lambda: adam(main)), "serial": timed(serial),
     "concurrent": timed(both)}
print(" ".join(f"{k} {v:.1f}" for k, v in r.items()), flush=True)
