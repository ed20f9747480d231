"""Path-tracing golden vectors from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden_pathtrace.py

The model / macro-cells of tests/golden/render_small.npz (loaded from its
.vnr-layout blob, no retraining) rendered in mode "pathtrace"
(_render_kernels.py:566-878) by the reference's wavefront driver at 48x27:
with and without macro-cells, frames 1 and 4, and on the dense grid field.
Writes tests/golden/render_pathtrace.npz (images + frame statistics).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from neuralvol import fields  # noqa: E402
from neuralvol.camera import default_camera  # noqa: E402
from neuralvol.macrocell import macrocell_build, macrocell_from_model, macrocell_set_tf  # noqa: E402
from neuralvol.model import build_model  # noqa: E402
from neuralvol.render import RenderConfig, render  # noqa: E402
from neuralvol.transfer import default_tf  # noqa: E402

GOLD = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main():
    z = np.load(GOLD / "render_small.npz")
    cfg = json.loads(str(z["config"]))
    dims = tuple(int(x) for x in z["dims"])
    model = build_model(cfg, dims=dims, seed=0)
    blob = z["blob"].astype(np.float32)
    k = model.encoder.params.size
    model.encoder.params[:] = blob[:k]
    pos = k
    for w in model.mlp.weights:
        w[...] = blob[pos:pos + w.size].reshape(w.shape)
        pos += w.size
    tf = default_tf()
    cam = default_camera(dims, 48, 27)
    grid = macrocell_from_model(model, n_g=8)
    macrocell_set_tf(grid, tf)
    assert np.array_equal(grid.mu_max, z["mc_mu"])
    fld = fields.rasterize("blobs", dims)
    gridf = macrocell_build(fld, n_g=8)
    macrocell_set_tf(gridf, tf)
    out = {}
    cases = {
        "pt_mc": (model, RenderConfig(mode="pathtrace", use_macrocells=True, seed=3), grid),
        "pt_nomc": (model, RenderConfig(mode="pathtrace", use_macrocells=False, seed=3), None),
        "pt_mc_f4": (model, RenderConfig(mode="pathtrace", use_macrocells=True, frames=4, seed=5, rr_depth=1), grid),
        "pt_grid_mc": (fld, RenderConfig(mode="pathtrace", use_macrocells=True, seed=7), gridf),
    }
    for name, (phi, rc, g) in cases.items():
        stats = []
        img = render(phi, tf, cam, rc, "wavefront", grid=g, stats_out=stats)
        out[f"img_{name}"] = img
        out[f"evals_{name}"] = np.array([s.evals for s in stats])
        out[f"viol_{name}"] = np.array([s.violations for s in stats])
        out[f"alive_{name}"] = np.array(stats[0].alive_per_iteration)
        print(name, "evals", [s.evals for s in stats], "iters", len(stats[0].alive_per_iteration), flush=True)
    np.savez_compressed(GOLD / "render_pathtrace.npz", **out)
    print("pathtrace golden written")


if __name__ == "__main__":
    main()
