"""Render / macro-cell golden vectors from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden_render.py

Writes tests/golden/render_*.npz: a small trained hash-grid model (as a .vnr
blob), the macro-cell grids the reference builds for it, and wavefront
renders (raymarch / raymarch_shadow, macro-cells on / off) with their frame
statistics.  Also a dense-grid (ScalarField) render.
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
from neuralvol.render import RenderConfig, render, render_reference  # noqa: E402
from neuralvol.sampler import InCoreSampler  # noqa: E402
from neuralvol.trainer import train  # noqa: E402
from neuralvol.transfer import default_tf  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

CFG = {"encoding": {"otype": "HashGrid", "n_levels": 8, "n_features_per_level": 2,
                    "log2_hashmap_size": 14, "base_resolution": 4},
       "network": {"n_neurons": 32, "n_hidden_layers": 2}, "batch_size": 16384}


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    dims = (40, 36, 32)
    fld = fields.rasterize("blobs", dims)
    model = build_model(CFG, dims=dims, seed=0)
    train(model, InCoreSampler(fld, seed=1), steps=60)
    blob = np.concatenate([model.encoder.params] + [w.ravel() for w in model.mlp.weights])
    tf = default_tf()
    cam = default_camera(dims, 48, 27)
    out = {"config": json.dumps(CFG), "dims": np.array(dims), "blob": blob}
    grid = macrocell_from_model(model, n_g=8)
    macrocell_set_tf(grid, tf)
    out.update(mc_lo=grid.value_lo, mc_hi=grid.value_hi, mc_mu=grid.mu_max)
    gridf = macrocell_build(fld, n_g=8)
    macrocell_set_tf(gridf, tf)
    out.update(mcf_lo=gridf.value_lo, mcf_hi=gridf.value_hi, mcf_mu=gridf.mu_max, norm=fld.normalized)
    cases = {
        "rm_mc": RenderConfig(mode="raymarch", use_macrocells=True, k_batch=8),
        "rm_nomc": RenderConfig(mode="raymarch", use_macrocells=False, k_batch=8),
        "rms_mc": RenderConfig(mode="raymarch_shadow", use_macrocells=True, k_batch=4),
        "rm_mc_step": RenderConfig(mode="raymarch", use_macrocells=True, k_batch=8, step_size=0.5, max_step=16.0),
    }
    for name, rc in cases.items():
        stats = []
        img = render(model, tf, cam, rc, "wavefront", grid=grid if rc.use_macrocells else None, stats_out=stats)
        out[f"img_{name}"] = img
        out[f"evals_{name}"] = stats[0].evals
        out[f"alive_{name}"] = np.array(stats[0].alive_per_iteration)
        print(name, "evals", stats[0].evals, "iters", len(stats[0].alive_per_iteration), flush=True)
    stats = []
    img = render(fld, tf, cam, RenderConfig(mode="raymarch", use_macrocells=True, k_batch=8), "wavefront",
                 grid=gridf, stats_out=stats)
    out["img_grid_mc"] = img
    out["evals_grid_mc"] = stats[0].evals
    stats = []
    ref = render_reference(model, tf, cam, RenderConfig(mode="raymarch", use_macrocells=True), grid=grid,
                           stats_out=stats)
    out["img_megakernel"] = ref
    np.savez_compressed(OUT / "render_small.npz", **out)
    print("render golden written")


if __name__ == "__main__":
    main()
