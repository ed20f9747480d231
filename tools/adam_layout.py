"""Adam's DRAM stream vs the layout of its state (timing only; build with
-DNVOL_ADAM_LAYOUT_EXPT=<layout>): 0 separate p / m / v arrays (the product), 1 m / v interleaved
in 8 KB blocks, 2 p / m / v interleaved in 8 KB blocks.  cfg2's 12,181,394 params; the gradient
either L2-resident (as in the step: written just before) or flushed."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_11620_b200 import _lib  # noqa: E402
from paper_2207_11620_b200.model import NAN_NONE  # noqa: E402

layout = int(sys.argv[1])
n = 12_181_394
P = torch.zeros(3 * n if layout == 2 else n, device="cuda")
G = torch.zeros(n, device="cuda")
M = torch.zeros(2 * n if layout == 1 else n, device="cuda")
V = torch.zeros(n, device="cuda")
for t in (P, G, M, V):
    assert t.data_ptr() % 128 == 0
sched = torch.tensor([0.005, 0.1, 0.001], dtype=torch.float32, device="cuda")
counter = torch.zeros(1, dtype=torch.int64, device="cuda")
ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
acc = torch.zeros(1, dtype=torch.float64, device="cuda")
ns = torch.tensor([NAN_NONE, 0], dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()


def adam():
    _lib.call("nvol_adam_train_step", _lib.ptr(P), _lib.ptr(G), _lib.ptr(M), _lib.ptr(V), n, _lib.ptr(sched), 1,
              _lib.ptr(counter), 0.9, 0.1, 0.999, 0.001, 1e-15, 1e-6, _lib.ptr(ns), _lib.ptr(acc), None, 0, 0, 1.0,
              _lib.ptr(ticket), main.cuda_stream)


def timed(g_resident, reps=40):
    ts = []
    for _ in range(reps):
        flush.add_(1)
        if g_resident:
            G.fill_(1e-3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        adam()
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for _ in range(3):
    adam()
a, b = timed(True), timed(False)
print(f"layout {layout}: g L2-resident {a:.1f} us ({6 * 4 * n / a / 1e3:.0f} GB/s on p/m/v)  flushed {b:.1f} us")
