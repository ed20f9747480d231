import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from conftest import golden, golden_config
from paper_2207_11620_b200 import macrocell
from paper_2207_11620_b200.camera import default_camera
from paper_2207_11620_b200.model import build_model
from paper_2207_11620_b200.render import RenderConfig, render
from paper_2207_11620_b200.transfer import default_tf
z = golden("render_small.npz"); g = golden("render_pathtrace.npz")
dims = tuple(int(x) for x in z["dims"])
model = build_model(golden_config(z), dims=dims, seed=0); model.load_blob(z["blob"])
grid = macrocell.macrocell_from_model(model, n_g=8); tf = default_tf(); macrocell.macrocell_set_tf(grid, tf)
cam = default_camera(dims, 48, 27)
for name, kw in {"pt_mc": dict(use_macrocells=True, seed=3), "pt_nomc": dict(use_macrocells=False, seed=3),
                 "pt_mc_f4": dict(use_macrocells=True, frames=4, seed=5, rr_depth=1)}.items():
    st = []
    img = render(model, tf, cam, RenderConfig(mode="pathtrace", **kw), "wavefront", grid=grid if kw["use_macrocells"] else None, stats_out=st)
    w = g[f"img_{name}"]
    print(name, "identical px", np.mean(np.all(img == w, axis=-1)), "maxdiff", np.abs(img - w).max(), "evals", [s.evals for s in st], list(g[f"evals_{name}"]))
