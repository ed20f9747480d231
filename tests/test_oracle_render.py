"""Pin the render / macro-cell oracle against the reference's golden renders (CPU)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_config


@pytest.fixture(scope="module")
def scene(oracle):
    import render_oracle as ro
    z = golden("render_small.npz")
    cfg = golden_config(z)
    dims = tuple(int(x) for x in z["dims"])
    model = oracle.OracleModel(cfg, seed=0)
    model.load_flat(z["blob"])
    return ro, z, model, dims


def test_macrocells_from_model_golden(scene):
    ro, z, model, dims = scene
    lo, hi = ro.macrocell_from_model(model, dims, 8)
    np.testing.assert_array_equal(lo, z["mc_lo"])
    np.testing.assert_array_equal(hi, z["mc_hi"])
    np.testing.assert_array_equal(ro.set_tf(lo, hi, ro.default_tf()), z["mc_mu"])


def test_macrocells_from_volume_golden(scene):
    ro, z, model, dims = scene
    lo, hi = ro.ranges_from_array(z["norm"], dims, 8)
    np.testing.assert_array_equal(lo, z["mcf_lo"])
    np.testing.assert_array_equal(hi, z["mcf_hi"])
    np.testing.assert_array_equal(ro.set_tf(lo, hi, ro.default_tf()), z["mcf_mu"])


CASES = {
    "rm_mc": dict(mode="raymarch", use_macrocells=True),
    "rm_nomc": dict(mode="raymarch", use_macrocells=False),
    "rms_mc": dict(mode="raymarch_shadow", use_macrocells=True, k_batch=4),
    "rm_mc_step": dict(mode="raymarch", use_macrocells=True, step_size=0.5, max_step=16.0),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_render_golden_bit_exact(scene, name):
    ro, z, model, dims = scene
    cam = ro.default_camera(dims, 48, 27)
    img, evals = ro.render(model, ro.default_tf(), cam, mu=z["mc_mu"], ng=8, dims=dims, **CASES[name])
    assert evals == int(z[f"evals_{name}"])
    np.testing.assert_array_equal(img, z[f"img_{name}"])


def test_render_grid_golden(scene):
    ro, z, model, dims = scene
    cam = ro.default_camera(dims, 48, 27)
    img, evals = ro.render(z["norm"], ro.default_tf(), cam, mu=z["mcf_mu"], ng=8, dims=dims)
    assert evals == int(z["evals_grid_mc"])
    np.testing.assert_array_equal(img, z["img_grid_mc"])


def test_online_macrocells_golden():
    """oracle update_online (macrocell.py:101-133) == the reference on its golden batches."""
    import render_oracle as ro
    z = golden("macrocell_online.npz")
    dims, ng = tuple(int(x) for x in z["dims"]), int(z["n_g"])
    gx, gy, gz = ro.grid_dims(dims, ng)
    lo = np.full((gz, gy, gx), np.inf, dtype=np.float32)
    hi = np.full((gz, gy, gx), -np.inf, dtype=np.float32)
    for c, t in zip(z["coords"], z["targets"]):
        ro.update_online(lo, hi, c, t, dims, ng)
    np.testing.assert_array_equal(lo, z["lo"])
    np.testing.assert_array_equal(hi, z["hi"])
