"""One 1080p cfg4 frame (wavefront, tensor evaluator) for ncu launch lists."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import CFG2, DIMS  # noqa: E402
from paper_2207_11620_b200 import fields  # noqa: E402
from paper_2207_11620_b200.camera import default_camera  # noqa: E402
from paper_2207_11620_b200.macrocell import macrocell_from_model, macrocell_set_tf  # noqa: E402
from paper_2207_11620_b200.model import build_model  # noqa: E402
from paper_2207_11620_b200.render import RenderConfig, render_frame_device  # noqa: E402
from paper_2207_11620_b200.sampler import InCoreSampler  # noqa: E402
from paper_2207_11620_b200.trainer import train  # noqa: E402
from paper_2207_11620_b200.transfer import default_tf  # noqa: E402

fld = fields.rasterize("blobs", DIMS)
m = build_model(CFG2, dims=DIMS, seed=0)
m.train_mode = 1
train(m, InCoreSampler(fld, seed=1), steps=300)
tf = default_tf()
grid = macrocell_from_model(m, n_g=16)
macrocell_set_tf(grid, tf)
cam = default_camera(DIMS, 1920, 1080)
cfg = RenderConfig(mode="raymarch", use_macrocells=True, k_batch=8, step_size=1.0, max_step=64.0)
mode = sys.argv[1] if len(sys.argv) > 1 else "tensor"
img, st = render_frame_device(m, tf, cam, cfg, grid, "wavefront", mode)
torch.cuda.synchronize()
torch.cuda.profiler.start()   # ncu --profile-from-start off: only this frame
img, st = render_frame_device(m, tf, cam, cfg, grid, "wavefront", mode)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("evals", st.evals, "iters", len(st.alive_per_iteration), st.alive_per_iteration)
