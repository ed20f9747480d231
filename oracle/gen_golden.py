"""Generate golden vectors from the REAL reference (run in the build container).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden.py [--psnr]

Writes small fixtures to tests/golden/.  The reference is imported read-only
from /root/reference (it does not exist on the GPU box); the fixtures travel
instead.  Every fixture records the reference call that produced it.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from neuralvol import _kernels, fields, network  # noqa: E402
from neuralvol.encoding import EncoderConfig, GridEncoder  # noqa: E402
from neuralvol.model import build_model  # noqa: E402
from neuralvol.network import OptimizerState, adam_step  # noqa: E402
from neuralvol.sampler import InCoreSampler  # noqa: E402
from neuralvol.trainer import decode, train  # noqa: E402
from neuralvol.volume import psnr  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

CFG1 = {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2,
                     "log2_hashmap_size": 12, "base_resolution": 4},
        "network": {"n_neurons": 16, "n_hidden_layers": 2}}
CFG2 = {"encoding": {"otype": "HashGrid", "n_levels": 16, "n_features_per_level": 2,
                     "log2_hashmap_size": 19, "base_resolution": 4},
        "network": {"n_neurons": 64, "n_hidden_layers": 4}}
ODD = {"encoding": {"otype": "HashGrid", "n_levels": 6, "n_features_per_level": 4,
                    "log2_hashmap_size": 10, "base_resolution": 5, "per_level_scale": 1.5},
       "network": {"n_neurons": 32, "n_hidden_layers": 1}}
DENSE = {"encoding": {"otype": "DenseGrid", "n_levels": 3, "n_features_per_level": 1,
                      "log2_hashmap_size": 10, "base_resolution": 3},
         "network": {"n_neurons": 16, "n_hidden_layers": 1, "output_activation": "None"}}
TINY = {"encoding": {"otype": "HashGrid", "n_levels": 2, "n_features_per_level": 2,
                     "log2_hashmap_size": 10, "base_resolution": 4},
        "network": {"n_neurons": 16, "n_hidden_layers": 1}, "batch_size": 512}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def edge_coords(rng, b):
    c = rng.random((b, 3)).astype(np.float32)
    one_below = np.nextafter(np.float32(1), np.float32(0))
    c[0] = 0.0
    c[1] = one_below
    c[2] = [0.5, 0.25, 0.125]           # lands exactly on lattice vertices
    c[3] = [one_below, 0.0, 0.5]
    c[4] = [1.0 / 3.0, 2.0 / 3.0, 0.999]
    return c


def encoder_fixture(name, cfg, b, seed=0, store_params=True):
    model = build_model(cfg, dims=(8, 8, 8), seed=seed)
    enc = model.encoder
    coords = edge_coords(np.random.default_rng(1234), b)
    feats, (idx, w) = model.encode_batch(coords)
    want = enc.encode(coords)
    # numba == numpy bitwise is what test_encoding.py:315-329 pins at cfg1; with
    # n_features_per_level == 1 numpy's einsum reorders the 8-corner sum, so
    # the numba kernel (the path the model uses) is the golden value.
    if enc.config.n_features_per_level > 1:
        assert np.array_equal(feats, want)
    dl = np.random.default_rng(99).normal(0, 1, feats.shape).astype(np.float32)
    grad = np.zeros_like(enc.params)
    _kernels.grid_encode_bwd(dl, idx, w, enc.config.n_features_per_level, grad)
    res, entries, dense, off = enc.kernel_tables()
    eval_fused = model.eval_fused(coords)
    eval_batch = model.eval_batch(coords)
    d = dict(config=json.dumps(cfg), seed=seed, coords=coords, idx_cache=idx.astype(np.int64),
             w_cache=w, feats=feats, dl_dfeat=dl, enc_grad=grad, res=res, entries=entries,
             dense=dense, offsets=off, numpy_encode=want, params_sha=sha(enc.params), eval_fused=eval_fused,
             eval_batch=eval_batch, weights_sha=sha(np.concatenate([x.ravel() for x in model.mlp.weights])))
    if store_params:
        d["params"] = enc.params
    np.savez_compressed(OUT / f"encode_{name}.npz", **d)
    print("encode", name, feats.shape, "grad nnz", np.count_nonzero(grad))


def adam_fixture():
    rng = np.random.default_rng(5)
    n = 4099
    out = {}
    for t in (0, 1, 2500, 12999):
        opt = OptimizerState()
        opt.t = t
        p = rng.normal(0, 0.1, n).astype(np.float32)
        g = rng.normal(0, 1e-3, n).astype(np.float32)
        g[::7] = 0.0
        m = rng.normal(0, 1e-4, n).astype(np.float32)
        v = np.abs(rng.normal(0, 1e-6, n)).astype(np.float32)
        opt.m, opt.v = [m.copy()], [v.copy()]
        p1, g1 = p.copy(), g.copy()
        adam_step(opt, [p1], [g1])
        out.update({f"p_{t}": p, f"g_{t}": g, f"m_{t}": m, f"v_{t}": v,
                    f"p1_{t}": p1, f"m1_{t}": opt.m[0], f"v1_{t}": opt.v[0]})
    np.savez_compressed(OUT / "adam.npz", **out)
    print("adam")


def sampler_fixture():
    f = fields.rasterize("mlobb", (20, 14, 11))
    s = InCoreSampler(f, seed=1)
    batches = [s.sample(1001) for _ in range(3)]   # 3*1001 is odd: exercises the buffered u32 half
    s2 = InCoreSampler(f, seed=7)
    big = s2.sample(65536)
    np.savez_compressed(OUT / "sampler.npz", norm=f.normalized, dims=np.array(f.meta.dims),
                        coords=np.stack([b.coords for b in batches]),
                        targets=np.stack([b.targets for b in batches]),
                        big_coords_head=big.coords[:4096], big_targets_head=big.targets[:4096],
                        big_coords_sha=sha(big.coords), big_targets_sha=sha(big.targets))
    print("sampler")


def mlp_fixture(name, cfg, b):
    model = build_model(cfg, dims=(8, 8, 8), seed=3)
    coords = np.random.default_rng(17).random((b, 3)).astype(np.float32)
    targets = np.random.default_rng(18).random(b).astype(np.float32)
    feats, _ = model.encode_batch(coords)
    # move features off their tiny init so the MLP sees realistic activations
    feats = (feats * 1e3).astype(np.float32)
    pred, acts = model.mlp.forward(feats)
    loss, dl = network.loss_and_grad(pred, targets, "L1")
    dfeat = model.mlp.backward(acts, dl)
    d = dict(feats=feats, targets=targets, pred=pred, loss=loss, dl_dpred=dl, dl_dfeat=dfeat)
    for i, (w, g) in enumerate(zip(model.mlp.weights, model.mlp.grads)):
        d[f"W{i}"] = w
        d[f"dW{i}"] = g
    for i, a in enumerate(acts):
        d[f"act{i}"] = a
    np.savez_compressed(OUT / f"mlp_{name}.npz", **d)
    print("mlp", name)


def train_fixture(name, cfg, dims, field, steps, batch):
    cfg = dict(cfg, batch_size=batch)
    fld = fields.rasterize(field, dims)
    model = build_model(cfg, dims=dims, seed=0)
    init = np.concatenate([model.encoder.params] + [w.ravel() for w in model.mlp.weights])
    hist = train(model, InCoreSampler(fld, seed=1), steps=steps)
    final = np.concatenate([model.encoder.params] + [w.ravel() for w in model.mlp.weights])
    dec = decode(model, dims=dims, slab_z=5)
    fused = model.eval_fused(np.random.default_rng(3).random((2048, 3)).astype(np.float32))
    np.savez_compressed(OUT / f"train_{name}.npz", config=json.dumps(cfg), dims=np.array(dims),
                        field=field, steps=steps, init=init, final=final,
                        losses=np.array(hist.losses), decode=dec.data, psnr=psnr(fld, dec),
                        fused_coords=np.random.default_rng(3).random((2048, 3)).astype(np.float32),
                        fused=fused, t=model.opt.t)
    print("train", name, "psnr", psnr(fld, dec), "final loss", hist.losses[-1])


def psnr_fixture(steps=2000, seeds=(1, 2, 3, 4, 5)):
    cfg = dict(CFG1, batch_size=65536)
    fld = fields.rasterize("mlobb", (64, 64, 64))
    vals = []
    for s in seeds:
        model = build_model(cfg, dims=(64, 64, 64), seed=0)
        train(model, InCoreSampler(fld, seed=s), steps=steps)
        vals.append(psnr(fld, decode(model, dims=(64, 64, 64))))
        print("psnr seed", s, vals[-1], flush=True)
    (OUT / "psnr_cfg1_mlobb.json").write_text(json.dumps(
        {"config": cfg, "field": "mlobb", "dims": [64, 64, 64], "steps": steps, "model_seed": 0,
         "sampler_seeds": list(seeds), "psnr_db": vals, "mean": float(np.mean(vals)),
         "std": float(np.std(vals))}, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--psnr", action="store_true", help="also run the 5-seed 2000-step cfg1 ensemble (~15 min)")
    args = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    encoder_fixture("cfg1", CFG1, 1024)
    encoder_fixture("cfg2", CFG2, 256, store_params=False)
    encoder_fixture("odd", ODD, 512)
    encoder_fixture("dense", DENSE, 512)
    adam_fixture()
    sampler_fixture()
    mlp_fixture("cfg1", CFG1, 512)
    mlp_fixture("cfg2", CFG2, 512)
    train_fixture("tiny", TINY, (16, 12, 10), "mlobb", 20, 512)
    train_fixture("cfg1", CFG1, (32, 32, 32), "mlobb", 30, 8192)
    if args.psnr:
        psnr_fixture()


if __name__ == "__main__":
    main()
