"""A few deterministic-mode cfg2 steps (eager) for an ncu launch list."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from bench import CFG2, DIMS, FIELD  # noqa: E402
from paper_2207_11620_b200 import encoding, fields  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402
from paper_2207_11620_b200.sampler import InCoreSampler  # noqa: E402
from paper_2207_11620_b200.trainer import StepPipeline  # noqa: E402
encoding.set_deterministic(True)
model = build_model(CFG2, dims=DIMS, seed=0)
pipe = StepPipeline(model, InCoreSampler(fields.rasterize(FIELD, DIMS), seed=1), capacity=4, use_graph=False)
pipe.step(2)
pipe.finish()
torch.cuda.synchronize()
