"""Deterministic-mode training rate at cfg2 (encoding.set_deterministic(True): fp32 SIMT engine with
ordered reductions) -- diagnostic; prints ms/step and checks two runs are bitwise identical."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from bench import CFG2, DIMS, FIELD  # noqa: E402
from paper_2207_11620_b200 import encoding, fields, trainer  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402
from paper_2207_11620_b200.sampler import InCoreSampler  # noqa: E402

encoding.set_deterministic(True)
fld = fields.rasterize(FIELD, DIMS)
out = []
for rep in range(2):
    m = build_model(CFG2, dims=DIMS, seed=0)
    trainer.train(m, InCoreSampler(fld, seed=1), steps=3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = trainer.train(m, InCoreSampler(fld, seed=1), steps=20)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    out.append((np.asarray(h.losses), m.flat_params.cpu().numpy()))
    print({"ms_per_step": dt * 1e3, "samples_per_s": 65536 / dt})
print({"bitwise_repeatable": bool(np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1]))})
