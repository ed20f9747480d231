"""GPU renderer / macro-cell parity against the reference's golden renders.

Bars: macro-cell ranges and majorants bit-exact (exact evaluator, float64
centres as macrocell.py:87-94); images: the reference composites with glibc
powf while the device evaluates pow in float64 and rounds (identical in all
but ~0.1% of inputs, 1 ulp), so images are compared at float tolerance
(max |diff| <= 2e-3, PSNR >= 50 dB) and field-evaluation counts within 1%;
schedule invariants (K batching, in-shader == wavefront) are bitwise.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import golden, golden_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene(nv):
    from paper_2207_11620_b200 import macrocell
    from paper_2207_11620_b200.camera import default_camera
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.transfer import default_tf
    z = golden("render_small.npz")
    dims = tuple(int(x) for x in z["dims"])
    model = build_model(golden_config(z), dims=dims, seed=0)
    model.load_blob(z["blob"])
    grid = macrocell.macrocell_from_model(model, n_g=8)
    tf = default_tf()
    macrocell.macrocell_set_tf(grid, tf)
    return z, dims, model, grid, tf, default_camera(dims, 48, 27)


def img_psnr(a, b):
    e = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return 99.0 if e == 0 else -10 * math.log10(e)


def test_macrocells_from_model_bit_exact(scene):
    z, dims, model, grid, tf, cam = scene
    np.testing.assert_array_equal(grid.value_lo.cpu().numpy(), z["mc_lo"])
    np.testing.assert_array_equal(grid.value_hi.cpu().numpy(), z["mc_hi"])
    np.testing.assert_array_equal(grid.mu_max.cpu().numpy(), z["mc_mu"])


def test_macrocells_from_volume_bit_exact(scene):
    from paper_2207_11620_b200 import macrocell
    from paper_2207_11620_b200.volume import ScalarField, VolumeMeta
    z, dims, model, grid, tf, cam = scene
    fld = ScalarField(VolumeMeta(dims, "f32", (0.0, 1.0)), z["norm"])
    g = macrocell.macrocell_build(fld, n_g=8)
    macrocell.macrocell_set_tf(g, tf)
    np.testing.assert_array_equal(g.value_lo.cpu().numpy(), z["mcf_lo"])
    np.testing.assert_array_equal(g.value_hi.cpu().numpy(), z["mcf_hi"])
    np.testing.assert_array_equal(g.mu_max.cpu().numpy(), z["mcf_mu"])


CASES = {
    "rm_mc": dict(mode="raymarch", use_macrocells=True),
    "rm_nomc": dict(mode="raymarch", use_macrocells=False),
    "rms_mc": dict(mode="raymarch_shadow", use_macrocells=True, k_batch=4),
    "rm_mc_step": dict(mode="raymarch", use_macrocells=True, step_size=0.5, max_step=16.0),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_wavefront_matches_reference(scene, name):
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    cfg = RenderConfig(**CASES[name])
    stats = []
    img = render(model, tf, cam, cfg, "wavefront", grid=grid if cfg.use_macrocells else None, stats_out=stats)
    want = z[f"img_{name}"]
    assert np.abs(img - want).max() <= 2e-3
    assert img_psnr(img, want) >= 50.0
    ev = int(z[f"evals_{name}"])
    assert abs(stats[0].evals - ev) <= max(2, 0.01 * ev)


def test_in_shader_equals_wavefront_and_reference(scene):
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    cfg = RenderConfig(mode="raymarch", use_macrocells=True)
    a = render(model, tf, cam, cfg, "reference", grid=grid)
    b = render(model, tf, cam, cfg, "wavefront", grid=grid)
    np.testing.assert_array_equal(a, b)                 # same device state machine, bitwise
    assert img_psnr(a, z["img_megakernel"]) >= 50.0


@pytest.mark.parametrize("mode", ["raymarch", "raymarch_shadow"])
def test_tensor_in_shader_equals_tensor_wavefront(scene, mode):
    """The in-shader marcher on the tensor cores (rm_tc_kernel: rays march in place, each round's
    128 samples of a CTA evaluated as one tcgen05 tile) runs the reference's per-ray sequence
    sample -> Phi -> consume with the batched evaluator's values: the image equals the tensor
    wavefront's bit for bit, and it evaluates exactly the samples the rays consume (no samples
    staged past termination), i.e. no more than the wavefront and no fewer than K = 1."""
    from paper_2207_11620_b200.camera import default_camera
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    cam = default_camera(dims, 320, 180)
    model.infer_mode = "tensor"
    try:
        out = {}
        for arch, k in (("reference", 8), ("wavefront", 8), ("wavefront", 1)):
            st = []
            img = render(model, tf, cam, RenderConfig(mode=mode, use_macrocells=True, k_batch=k), arch, grid=grid,
                         stats_out=st)
            out[(arch, k)] = (img, st[0].evals)
    finally:
        model.infer_mode = "exact"
    np.testing.assert_array_equal(out[("reference", 8)][0], out[("wavefront", 8)][0])
    assert out[("reference", 8)][1] == out[("wavefront", 1)][1]
    assert out[("reference", 8)][1] <= out[("wavefront", 8)][1]


def test_k_batching_is_scheduling_only(scene):
    # test_render.py:116-128
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    imgs = [render(model, tf, cam, RenderConfig(mode="raymarch", use_macrocells=True, k_batch=k), grid=grid)
            for k in (1, 3, 8, 16)]
    for im in imgs[1:]:
        np.testing.assert_array_equal(im, imgs[0])


def test_macrocells_never_increase_evals(scene):
    # test_render.py:234-255
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    s_on, s_off = [], []
    render(model, tf, cam, RenderConfig(mode="raymarch", use_macrocells=True), "reference", grid=grid, stats_out=s_on)
    render(model, tf, cam, RenderConfig(mode="raymarch", use_macrocells=False), "reference", stats_out=s_off)
    assert s_on[0].evals <= s_off[0].evals


def test_grid_field_render(scene):
    from paper_2207_11620_b200 import macrocell
    from paper_2207_11620_b200.render import RenderConfig, render
    from paper_2207_11620_b200.volume import ScalarField, VolumeMeta
    z, dims, model, grid, tf, cam = scene
    fld = ScalarField(VolumeMeta(dims, "f32", (0.0, 1.0)), z["norm"])
    g = macrocell.macrocell_build(fld, n_g=8)
    stats = []
    img = render(fld, tf, cam, RenderConfig(mode="raymarch", use_macrocells=True), grid=g, stats_out=stats)
    assert np.abs(img - z["img_grid_mc"]).max() <= 2e-3
    assert abs(stats[0].evals - int(z["evals_grid_mc"])) <= max(2, 0.01 * int(z["evals_grid_mc"]))


def test_tensor_core_batched_inference_render(scene):
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    model.infer_mode = "tensor"
    try:
        img = render(model, tf, cam, RenderConfig(mode="raymarch", use_macrocells=True), "wavefront", grid=grid)
    finally:
        model.infer_mode = "exact"
    assert img_psnr(img, z["img_rm_mc"]) >= 35.0


def test_tensor_wavefront_schedule_is_scheduling_only(scene):
    """The host-sync-free tensor wavefront (device counts, one-iteration-late bounds) gives
    the same image, evaluation count and per-iteration alive counts as the synchronous
    loop, bitwise, and K batching changes nothing in the image."""
    import ast
    import subprocess
    import sys
    from paper_2207_11620_b200.camera import default_camera
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    cam = default_camera(dims, 320, 180)
    model.infer_mode = "tensor"
    try:
        runs = {}
        for k in (1, 3, 8):
            st = []
            img = render(model, tf, cam, RenderConfig(mode="raymarch", use_macrocells=True, k_batch=k), "wavefront",
                         grid=grid, stats_out=st)
            runs[k] = (img, st[0])
    finally:
        model.infer_mode = "exact"
    for k in (3, 8):   # (evaluation counts do depend on K: samples staged past termination are evaluated)
        np.testing.assert_array_equal(runs[k][0], runs[1][0])
    # the synchronous loop (NVOL_RENDER_SYNC=1 is read once per process: run it in a child)
    code = (
        "import sys, numpy as np; sys.path.insert(0, 'tests'); from conftest import golden, golden_config\n"
        "from paper_2207_11620_b200 import macrocell\n"
        "from paper_2207_11620_b200.camera import default_camera\n"
        "from paper_2207_11620_b200.model import build_model\n"
        "from paper_2207_11620_b200.render import RenderConfig, render\n"
        "from paper_2207_11620_b200.transfer import default_tf\n"
        "z = golden('render_small.npz'); dims = tuple(int(x) for x in z['dims'])\n"
        "m = build_model(golden_config(z), dims=dims, seed=0); m.load_blob(z['blob'])\n"
        "g = macrocell.macrocell_from_model(m, n_g=8); tf = default_tf(); macrocell.macrocell_set_tf(g, tf)\n"
        "m.infer_mode = 'tensor'; st = []\n"
        "img = render(m, tf, default_camera(dims, 320, 180), RenderConfig(mode='raymarch', use_macrocells=True),"
        " 'wavefront', grid=g, stats_out=st)\n"
        "np.save(sys.argv[1], img); print(st[0].evals, list(st[0].alive_per_iteration))\n")
    import os
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "img.npy")
        env = dict(os.environ, NVOL_RENDER_SYNC="1")
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code, out], env=env, cwd=root, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        ev, hist = r.stdout.strip().splitlines()[-1].split(" ", 1)
        np.testing.assert_array_equal(np.load(out), runs[8][0])
        assert int(ev) == runs[8][1].evals
        assert ast.literal_eval(hist) == list(runs[8][1].alive_per_iteration)


def test_online_macrocells_inside_precomputed(nv):
    # test_macrocell.py:116-139: streamed ranges never exceed the bordered precomputed ones
    from paper_2207_11620_b200 import fields, macrocell
    from paper_2207_11620_b200.sampler import InCoreSampler
    fld = fields.rasterize("blobs", (24, 20, 16), host=True)
    pre = macrocell.macrocell_build(fld, n_g=4)
    onl = macrocell.macrocell_empty((24, 20, 16), n_g=4)
    s = InCoreSampler(fld, seed=3)
    for _ in range(20):
        macrocell.macrocell_update_online(onl, s.sample(4096))
    lo, hi = onl.value_lo.cpu().numpy(), onl.value_hi.cpu().numpy()
    plo, phi = pre.value_lo.cpu().numpy(), pre.value_hi.cpu().numpy()
    touched = lo <= hi
    assert touched.mean() > 0.9
    assert np.all(lo[touched] >= plo[touched] - 1e-7) and np.all(hi[touched] <= phi[touched] + 1e-7)


def test_online_macrocells_bit_exact(nv):
    """nvol_macrocell_update_online on the reference's golden batches == the reference."""
    from paper_2207_11620_b200 import macrocell
    from paper_2207_11620_b200.sampler import SampleBatch
    z = golden("macrocell_online.npz")
    dims, ng = tuple(int(x) for x in z["dims"]), int(z["n_g"])
    grid = macrocell.macrocell_empty(dims, n_g=ng)
    for c, t in zip(z["coords"], z["targets"]):
        macrocell.macrocell_update_online(grid, SampleBatch(c, t))
    np.testing.assert_array_equal(grid.value_lo.cpu().numpy(), z["lo"])
    np.testing.assert_array_equal(grid.value_hi.cpu().numpy(), z["hi"])


def test_online_macrocells_fused_into_training(nv):
    """train(..., tap=OnlineMacrocells(grid)) fuses the update into the device sampler:
    after 5 steps the grid equals the reference's update over the same 5 batches."""
    from paper_2207_11620_b200 import fields, macrocell, trainer
    from paper_2207_11620_b200.model import MODE_TCGEN05, build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    z = golden("macrocell_online.npz")
    dims, ng = tuple(int(x) for x in z["dims"]), int(z["n_g"])
    fld = fields.rasterize("blobs", dims, host=True)
    cfg = {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2,
                        "log2_hashmap_size": 12, "base_resolution": 4},
           "network": {"n_neurons": 16, "n_hidden_layers": 2}, "batch_size": 4096}
    for mode in (0, MODE_TCGEN05):
        model = build_model(cfg, dims=dims, seed=0)
        model.train_mode = mode
        grid = macrocell.macrocell_empty(dims, n_g=ng)
        trainer.train(model, InCoreSampler(fld, seed=3), steps=5, tap=macrocell.OnlineMacrocells(grid))
        np.testing.assert_array_equal(grid.value_lo.cpu().numpy(), z["lo"])
        np.testing.assert_array_equal(grid.value_hi.cpu().numpy(), z["hi"])


def test_render_tiles_assemble_bit_identically(scene):
    """distributed.render_tile: image tiles of 3 (virtual) ranks == the full frame, bitwise,
    and their evaluation counts add up (rays are independent)."""
    from paper_2207_11620_b200.distributed import render_tile
    from paper_2207_11620_b200.render import RenderConfig, render_frame_device
    z, dims, model, grid, tf, cam = scene
    cfg = RenderConfig(mode="raymarch", use_macrocells=True, k_batch=8)
    for emode in ("exact", "tensor"):
        full, st = render_frame_device(model, tf, cam, cfg, grid, "wavefront", emode)
        parts, evals = [], 0
        for r in range(3):
            row0, tile, s = render_tile(model, tf, cam, cfg, grid, rank=r, world=3, eval_mode=emode)
            parts.append(tile)
            evals += s.evals
        assert torch.equal(torch.cat(parts), full)
        assert evals == st.evals


# ----------------------------------------------------------------------------- path tracing (SURVEY 8 f item 3)

PT_CASES = {
    "pt_mc": dict(mode="pathtrace", use_macrocells=True, seed=3),
    "pt_nomc": dict(mode="pathtrace", use_macrocells=False, seed=3),
    "pt_mc_f4": dict(mode="pathtrace", use_macrocells=True, frames=4, seed=5, rr_depth=1),
}


@pytest.mark.parametrize("name", sorted(PT_CASES))
def test_pathtrace_matches_reference(scene, name):
    """Wavefront path tracer (exact evaluator) vs the reference's renders
    (oracle/gen_golden_pathtrace.py): the counter RNG, the tracking arithmetic
    (float64 / float32 in the reference's order) and the f32 casts follow the
    reference, and the images and per-frame field-evaluation counts come out
    bit-identical on these scenes (the device's float64 log1p / cos / sin agree
    with glibc's to the bit here; an ulp difference could flip a rare
    Monte-Carlo decision, which would show up as a failure of this bar)."""
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    g = golden("render_pathtrace.npz")
    cfg = RenderConfig(**PT_CASES[name])
    stats = []
    model.infer_mode = "exact"
    img = render(model, tf, cam, cfg, "wavefront", grid=grid if cfg.use_macrocells else None, stats_out=stats)
    np.testing.assert_array_equal(img, g[f"img_{name}"])
    np.testing.assert_array_equal([s.evals for s in stats], g[f"evals_{name}"])
    np.testing.assert_array_equal([s.violations for s in stats], g[f"viol_{name}"])


def test_pathtrace_grid_field_matches_reference(scene):
    from paper_2207_11620_b200 import fields, macrocell
    from paper_2207_11620_b200.render import RenderConfig, render
    z, dims, model, grid, tf, cam = scene
    g = golden("render_pathtrace.npz")
    fld = fields.rasterize("blobs", dims, host=True)
    gridf = macrocell.macrocell_build(fld, n_g=8)
    macrocell.macrocell_set_tf(gridf, tf)
    img = render(fld, tf, cam, RenderConfig(mode="pathtrace", use_macrocells=True, seed=7), "wavefront", grid=gridf)
    np.testing.assert_array_equal(img, g["img_pt_grid_mc"])


def test_pathtrace_wavefront_equals_megakernel(scene):
    """render_wavefront == render_reference bitwise for the path tracer, as the
    reference's own test (test_render.py:90-113): same per-ray state machine,
    one collision per wavefront iteration."""
    from paper_2207_11620_b200.render import RenderConfig, render_reference, render_wavefront
    z, dims, model, grid, tf, cam = scene
    model.infer_mode = "exact"
    for mc in (True, False):
        cfg = RenderConfig(mode="pathtrace", use_macrocells=mc, seed=11)
        s1, s2 = [], []
        a = render_wavefront(model, tf, cam, cfg, grid=grid if mc else None, stats_out=s1)
        b = render_reference(model, tf, cam, cfg, grid=grid if mc else None, stats_out=s2)
        np.testing.assert_array_equal(a, b)
        assert s1[0].evals == s2[0].evals
        assert s1[0].violations == s2[0].violations


def test_macrocell_from_model_duck_typed(nv):
    """macrocell_from_model accepts any object with the reference's dims + eval_fused protocol
    (macrocell.py:84-98; the reference's test_macrocell.py::test_from_model_axis_order)."""
    from paper_2207_11620_b200.macrocell import macrocell_from_model

    class Stub:
        dims = (6, 4, 5)

        def eval_fused(self, coords):
            return coords[:, 0].astype(np.float32)  # value = x coordinate

    g = macrocell_from_model(Stub(), n_g=2, chunk=17)
    lo, hi = g.value_lo.cpu().numpy(), g.value_hi.cpu().numpy()
    for cx in range(3):
        assert np.allclose(lo[:, :, cx], np.float32((max(2 * cx - 1, 0) + 0.5) / 6))
        assert np.allclose(hi[:, :, cx], np.float32((min(2 * cx + 2, 5) + 0.5) / 6))
