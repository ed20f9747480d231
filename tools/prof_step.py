"""Run a few cfg2 training steps (eager, no graph) for ncu captures.

    python tools/prof_step.py [--mode 1] [--steps 3] [--decode N]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import CFG2, DIMS, FIELD  # noqa: E402
from paper_2207_11620_b200 import fields  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402
from paper_2207_11620_b200.sampler import InCoreSampler  # noqa: E402
from paper_2207_11620_b200.trainer import StepPipeline, decode  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", type=int, default=1)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--decode", type=int, default=0)
ap.add_argument("--decode-mode", default="exact")
a = ap.parse_args()
model = build_model(CFG2, dims=DIMS, seed=0)
model.train_mode = a.mode
field = fields.rasterize(FIELD, DIMS)
pipe = StepPipeline(model, InCoreSampler(field, seed=1), capacity=a.steps + 1, use_graph=False)
pipe.step(a.steps)
print("losses", pipe.finish())
if a.decode:
    model.infer_mode = a.decode_mode
    decode(model, dims=(a.decode,) * 3)
torch.cuda.synchronize()
