"""CTA-0 timeline of mlp_tc4_kernel (library built with EXTRA=-DNVOL_TIMELINE)."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CFG2, DIMS, FIELD  # noqa: E402
from paper_2207_11620_b200 import _lib, fields  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402
from paper_2207_11620_b200.sampler import InCoreSampler  # noqa: E402
from paper_2207_11620_b200.trainer import StepPipeline  # noqa: E402

model = build_model(CFG2, dims=DIMS, seed=0)
model.train_mode = 1
field = fields.rasterize(FIELD, DIMS)
pipe = StepPipeline(model, InCoreSampler(field, seed=1), capacity=4, use_graph=False)
pipe.step(3)
torch.cuda.synchronize()
lib = _lib.open_library()
buf = (ctypes.c_ulonglong * 4096)()
lib.nvol_debug_timeline(buf, 4096)
a = np.array(buf[:], dtype=np.uint64)
t0, t1 = int(a[4000]), int(a[4001])
e0, fl = int(a[4002]), int(a[4003])
print(f"CTA0: entry -> MMA warp start {(t0 - e0) / 1e3:.2f} us (prologue), MMA start -> flush {(fl - t0) / 1e3:.2f} us, "
      f"flush -> end {(t1 - fl) / 1e3:.2f} us, total {(t1 - e0) / 1e3:.2f} us")
print(f"CTA0 kernel span (MMA warp start -> end) {(t1 - t0) / 1e3:.2f} us")
mask = (1 << 52) - 1
for k in range(200):
    s, c = int(a[2 * k]), int(a[2 * k + 1])
    if s == 0:
        break
    t, ph = c >> 60, (c >> 52) & 0xFF
    print(f"mma {k:2d} slot {t} ph {ph:2d}: issue {(s - t0) / 1e3:7.2f}  issued {((c & mask) - (t0 & mask)) / 1e3:7.2f}")
for t in range(4):
    for k in range(0, 40):
        w, r = int(a[1024 + t * 256 + 2 * k]), int(a[1024 + t * 256 + 2 * k + 1])
        if w == 0:
            break
        print(f"slot {t} epi {k:2d}: acc-ready {(w - t0) / 1e3:7.2f}  release {(r - t0) / 1e3 if r else -1:7.2f}")
for t in range(4):
    m = [int(a[3000 + t * 8 + i]) for i in range(4)]
    if m[0]:
        print(f"slot {t} last fwd epilogue: start {(m[0] - t0) / 1e3:7.2f}  fence+sync {(m[1] - m[0]) / 1e3:5.2f}  "
              f"output dot {(m[2] - m[1]) / 1e3:5.2f}  loss {(m[3] - m[2]) / 1e3:5.2f}")
for t in range(2):
    for e in range(8):
        w = [int(a[3200 + t * 64 + e * 4 + q]) for q in range(4)]
        if w[0]:
            print(f"slot {t} epi {e}: warp releases " + " ".join(f"{(x - t0) / 1e3:7.2f}" for x in w))
fl0 = int(a[4003])
if fl0:
    w1 = [int(a[3600 + w]) for w in range(18)]
    print("flush, per warp (us after the flush start): dW out " +
          " ".join(f"{(x - fl0) / 1e3:.2f}" if x else "-" for x in w1))
