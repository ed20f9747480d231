"""Accuracy + speed of the tcgen05 (split-fp16) evaluator vs the exact one."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import golden, golden_config  # noqa: E402
from paper_2207_11620_b200 import trainer  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402


def rel_err(a, b, floor):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor * np.max(np.abs(b)))))


for name in ("cfg1", "cfg2", "odd"):
    z = golden(f"encode_{name}.npz")
    model = build_model(golden_config(z), dims=(20, 16, 12), seed=0)
    r = np.random.default_rng(2)
    model.encoder.params.copy_(torch.from_numpy(r.normal(0, 0.3, model.encoder.params.shape).astype(np.float32)))
    c = r.random((5000, 3)).astype(np.float32)
    ex = model.eval_fused(c)
    tc = model.eval_device(torch.from_numpy(c).cuda(), "tensor").cpu().numpy()
    print(name, "rel err (floor 1e-2)", rel_err(tc, ex, 1e-2), "(floor 1e-3)", rel_err(tc, ex, 1e-3))

from bench import CFG2, DIMS  # noqa: E402
m = build_model(CFG2, dims=DIMS, seed=0)
m.infer_mode = "tensor"
trainer.decode(m, dims=(64, 64, 64))
torch.cuda.synchronize()
for n in (256, 512):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    trainer.decode(m, dims=(n, n, n))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"decode {n}^3: {ms:.2f} ms  {n ** 3 / ms / 1e6:.3f} G samples/s")
