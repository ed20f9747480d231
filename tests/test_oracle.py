"""Pin the CPU oracle against the reference's own golden vectors (CPU-only).

Fixtures in tests/golden/ were produced by oracle/gen_golden.py, which imports
the real reference (/root/reference/pkg/src/neuralvol) in the build container.
Known answers restate the reference tests cited beside each case.
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden, golden_config


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- known answers (reference tests)

def test_level_tables_known_answers(oracle):
    # test_encoding.py:74-83 level_resolution examples
    spec = oracle.GridSpec(n_levels=4, n_features_per_level=1, log2_hashmap_size=15, base_resolution=4)
    res, entries, dense, off = oracle.level_tables(spec)
    assert res[0] == 4 and res[3] == 32
    spec = oracle.GridSpec(n_levels=3, base_resolution=16, per_level_scale=1.5)
    assert oracle.level_tables(spec)[0][2] == 36
    # SURVEY §8 cfg1 / cfg2 parameter counts
    c1 = oracle.GridSpec(n_levels=4, n_features_per_level=2, log2_hashmap_size=12, base_resolution=4)
    r, e, d, o = oracle.level_tables(c1)
    assert list(e) == [125, 729, 4096, 4096] and int((e * 2).sum()) == 18092
    assert list(d) == [1, 1, 0, 0]
    c2 = oracle.GridSpec(n_levels=16, n_features_per_level=2, log2_hashmap_size=19, base_resolution=4)
    assert int((oracle.level_tables(c2)[1] * 2).sum()) == 12166994


def test_dense_known_answer(oracle):
    # test_encoding.py:143-158: dense R=2 grid, params = vertex x -> 0.6
    spec = oracle.GridSpec(kind="densegrid", n_levels=1, n_features_per_level=1, base_resolution=2)
    vals = np.zeros(27, dtype=np.float32)
    for z in range(3):
        for y in range(3):
            for x in range(3):
                vals[(z * 3 + y) * 3 + x] = x
    out, idx, w = oracle.grid_encode_fwd(np.array([[0.3, 0.6, 0.9]], np.float32), vals, spec)
    assert out[0, 0] == pytest.approx(0.6, abs=1e-6)
    # test_encoding.py:91-95 dense row-major slots 86 / 0 / 124 (R=4): vertex (1,2,3) -> 86
    spec4 = oracle.GridSpec(kind="densegrid", n_levels=1, n_features_per_level=1, base_resolution=4)
    p = np.array([[1 / 4 + 1e-3, 2 / 4 + 1e-3, 3 / 4 + 1e-3]], np.float32)
    _, idx, _ = oracle.grid_encode_fwd(p, np.zeros(125, np.float32), spec4)
    assert idx[0, 0, 0] == 86


def test_border_clamp_known_answer(oracle):
    # test_encoding.py:161-170: p -> 1, cell clamps to R-1, approaches vertex value 26
    spec = oracle.GridSpec(kind="densegrid", n_levels=1, n_features_per_level=1, base_resolution=2)
    out, _, _ = oracle.grid_encode_fwd(np.full((1, 3), 0.999999, np.float32),
                                       np.arange(27, dtype=np.float32), spec)
    assert out[0, 0] == pytest.approx(26.0, abs=1e-3)


def test_adam_first_step_known_answer(oracle):
    # test_network.py:254-261: lone parameter moves by exactly -lr on step 1
    opt = oracle.AdamState(l2_reg=0.0)
    p, g = np.zeros(1, np.float32), np.array([0.37], np.float32)
    oracle.adam_step(opt, [p], [g])
    assert p[0] == pytest.approx(-0.005, rel=1e-6) and g[0] == 0.0 and opt.t == 1


def test_lr_schedule_known_answers(oracle):
    # test_network.py:220-227
    opt = oracle.AdamState()
    assert oracle.lr_at(opt, 0) == 0.005 and oracle.lr_at(opt, 2999) == 0.005
    assert oracle.lr_at(opt, 3000) == pytest.approx(0.005 * 0.99)
    assert oracle.lr_at(opt, 12999) == pytest.approx(0.005 * 0.99 ** 10)


def test_adam_nan_location(oracle):
    # test_network.py:282-288
    opt = oracle.AdamState()
    p1, p2 = np.zeros(4, np.float32), np.zeros((2, 3), np.float32)
    g1, g2 = np.zeros(4, np.float32), np.zeros((2, 3), np.float32)
    g2[1, 2] = np.nan
    with pytest.raises(FloatingPointError, match=r"group 1.*flat index 5"):
        oracle.adam_step(opt, [p1, p2], [g1, g2])


# ---------------------------------------------------------------- golden vectors (bit-exact)

@pytest.mark.parametrize("name", ["cfg1", "cfg2", "odd", "dense"])
def test_encoder_fwd_bwd_golden(oracle, name):
    z = golden(f"encode_{name}.npz")
    cfg = golden_config(z)
    model = oracle.OracleModel(cfg, seed=int(z["seed"]))
    assert _sha(model.params) == str(z["params_sha"])
    r, e, d, o = oracle.level_tables(model.spec)
    np.testing.assert_array_equal(r, z["res"])
    np.testing.assert_array_equal(e, z["entries"])
    np.testing.assert_array_equal(d, z["dense"])
    np.testing.assert_array_equal(o, z["offsets"])
    feats, idx, w = model.encode_batch(z["coords"])
    np.testing.assert_array_equal(idx, z["idx_cache"])         # slots: bit-exact
    np.testing.assert_array_equal(w, z["w_cache"])             # corner weights: bit-exact
    np.testing.assert_array_equal(feats, z["feats"])           # encodings: bit-exact
    grad = np.zeros_like(model.params)
    oracle.grid_encode_bwd(z["dl_dfeat"], idx, w, model.spec.n_features_per_level, grad)
    np.testing.assert_array_equal(grad, z["enc_grad"])         # serial scatter order kept
    np.testing.assert_array_equal(model.eval_fused(z["coords"]), z["eval_fused"])
    np.testing.assert_allclose(model.eval_batch(z["coords"]), z["eval_batch"], rtol=1e-5, atol=1e-7)


def test_adam_golden(oracle):
    z = golden("adam.npz")
    for t in (0, 1, 2500, 12999):
        opt = oracle.AdamState(t=t)
        p, g = z[f"p_{t}"].copy(), z[f"g_{t}"].copy()
        opt.m, opt.v = [z[f"m_{t}"].copy()], [z[f"v_{t}"].copy()]
        oracle.adam_step(opt, [p], [g])
        np.testing.assert_array_equal(p, z[f"p1_{t}"])
        np.testing.assert_array_equal(opt.m[0], z[f"m1_{t}"])
        np.testing.assert_array_equal(opt.v[0], z[f"v1_{t}"])
        assert not g.any()


def test_pcg64_matches_numpy(oracle):
    for seed in (0, 1, 7, 123456789):
        want = np.random.default_rng(seed).random(10001, dtype=np.float32)
        np.testing.assert_array_equal(oracle.pcg64_random_f32(seed, 0, 10001), want)
        np.testing.assert_array_equal(oracle.pcg64_random_f32(seed, 3, 9998), want[3:])
        np.testing.assert_array_equal(oracle.pcg64_random_f32(seed, 4000, 77), want[4000:4077])


def test_sampler_golden(oracle):
    z = golden("sampler.npz")
    s = oracle.InCoreSampler(z["norm"], seed=1)
    for k in range(3):
        c, t = s.sample(1001)
        np.testing.assert_array_equal(c, z["coords"][k])
        np.testing.assert_array_equal(t, z["targets"][k])
    s2 = oracle.InCoreSampler(z["norm"], seed=7)
    c, t = s2.sample(65536)
    assert _sha(c) == str(z["big_coords_sha"]) and _sha(t) == str(z["big_targets_sha"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_mlp_golden(oracle, name):
    z = golden(f"mlp_{name}.npz")
    nl = sum(1 for k in z.files if k.startswith("W"))
    weights = [z[f"W{i}"] for i in range(nl)]
    pred, acts = oracle.mlp_forward(z["feats"], weights)
    np.testing.assert_array_equal(pred, z["pred"])   # same numpy/OpenBLAS calls as the reference
    loss, dl = oracle.loss_and_grad(pred, z["targets"])
    assert loss == float(z["loss"])
    np.testing.assert_array_equal(dl, z["dl_dpred"])
    grads = [np.zeros_like(w) for w in weights]
    dfeat = oracle.mlp_backward(acts, weights, grads, dl)
    np.testing.assert_allclose(dfeat, z["dl_dfeat"], rtol=1e-6, atol=1e-12)
    for i in range(nl):
        np.testing.assert_allclose(grads[i], z[f"dW{i}"], rtol=1e-5, atol=1e-10)


@pytest.mark.parametrize("name", ["tiny", "cfg1"])
def test_train_golden(oracle, name):
    z = golden(f"train_{name}.npz")
    cfg = golden_config(z)
    dims = tuple(int(x) for x in z["dims"])
    model = oracle.OracleModel(cfg, seed=0)
    np.testing.assert_array_equal(model.flat_params(), z["init"])
    norm = oracle.rasterize(str(z["field"]), dims)
    s = oracle.InCoreSampler(norm, seed=1)
    losses = []
    for _ in range(int(z["steps"])):
        c, t = s.sample(model.batch_size)
        losses.append(model.train_step(c, t))
    np.testing.assert_allclose(losses, z["losses"], rtol=1e-6)
    np.testing.assert_allclose(model.flat_params(), z["final"], rtol=1e-4, atol=1e-6)
    dec = oracle.decode(model, dims, slab_z=5)
    np.testing.assert_allclose(dec, z["decode"], rtol=1e-4, atol=1e-5)
    assert oracle.psnr(norm, dec) == pytest.approx(float(z["psnr"]), abs=1e-3)
