"""Parity fixtures at the bench's own inference configs (cfg3 decode, cfg4 render) -- test
infrastructure, run in the build container (the reference is imported read-only).

    OPENBLAS_NUM_THREADS=1 python oracle/gen_golden_cfg34.py

The reference (/root/reference/pkg/src/neuralvol) trains its cfg2 model (HashGrid 16 x 2^19 x 2,
4 x 64 MLP) 300 steps on blobs 256^3 (the cfg4 scene), writes it with
trainer.save_model -> tests/golden_big/cfg2_blobs.vnr (48.7 MB: git-ignored, travels to the GPU
box with the repo snapshot; its sha256 is recorded in the committed fixture), then records
  * macrocell_from_model(model, n_g=16) + macrocell_set_tf(default_tf())   (macrocell.py:77-156)
  * render(model, default_tf(), default_camera(dims, 192, 108), RenderConfig(mode="raymarch",
    use_macrocells=True, k_batch=8, step_size=1, max_step=64), "wavefront", grid)  (render.py:383-454)
    -- the cfg4 frame at 192x108 (SURVEY §8(c) render protocol)
  * the cfg3 decode of a 64^3 window of the 1024^3 grid: eval_batch (decode_slabs' path,
    trainer.py:80-106) and eval_fused at those voxel centres
into tests/golden/cfg34.npz.
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from neuralvol import fields  # noqa: E402
from neuralvol.camera import default_camera  # noqa: E402
from neuralvol.macrocell import macrocell_from_model, macrocell_set_tf  # noqa: E402
from neuralvol.model import build_model  # noqa: E402
from neuralvol.render import RenderConfig, render  # noqa: E402
from neuralvol.sampler import InCoreSampler  # noqa: E402
from neuralvol.trainer import save_model, train  # noqa: E402
from neuralvol.transfer import default_tf  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
CFG2 = {"encoding": {"otype": "HashGrid", "n_levels": 16, "n_features_per_level": 2,
                     "log2_hashmap_size": 19, "base_resolution": 4},
        "network": {"n_neurons": 64, "n_hidden_layers": 4}, "batch_size": 65536}
DIMS = (256, 256, 256)
W0, WN, D = 480, 64, 1024          # decode window [480, 544)^3 of the 1024^3 grid


def main():
    (ROOT / "tests" / "golden_big").mkdir(exist_ok=True)
    fld = fields.rasterize("blobs", DIMS)
    m = build_model(CFG2, dims=DIMS, seed=0)
    train(m, InCoreSampler(fld, seed=1), steps=300)
    vnr = ROOT / "tests" / "golden_big" / "cfg2_blobs.vnr"
    save_model(m, vnr)
    sha = hashlib.sha256(vnr.read_bytes()).hexdigest()
    print("model written", sha, flush=True)
    tf = default_tf()
    grid = macrocell_from_model(m, n_g=16)
    macrocell_set_tf(grid, tf)
    print("macrocells done", flush=True)
    cam = default_camera(DIMS, 192, 108)
    rc = RenderConfig(mode="raymarch", use_macrocells=True, k_batch=8, step_size=1.0, max_step=64.0)
    stats = []
    img = render(m, tf, cam, rc, "wavefront", grid=grid, stats_out=stats)
    print("render done: evals", stats[0].evals, flush=True)
    ax = (np.arange(W0, W0 + WN, dtype=np.float32) + np.float32(0.5)) / np.float32(D)
    gz, gy, gx = np.meshgrid(ax, ax, ax, indexing="ij")
    coords = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    dec_batch = m.eval_batch(coords).reshape(WN, WN, WN)
    dec_fused = m.eval_fused(coords).reshape(WN, WN, WN)
    np.savez_compressed(ROOT / "tests" / "golden" / "cfg34.npz", vnr_sha256=sha, mc_lo=grid.value_lo,
                        mc_hi=grid.value_hi, mc_mu=grid.mu_max, img=img, evals=stats[0].evals,
                        alive=np.array(stats[0].alive_per_iteration), window=np.array([W0, WN, D]),
                        decode_batch=dec_batch, decode_fused=dec_fused)
    print("fixture written")


if __name__ == "__main__":
    main()
