"""The reference's acceptance gate 3 on the device (main arm).

/root/reference/pkg/tests/test_acceptance.py:186-233 (`test_3_hash_grid_convergence`) trains the
~1 M-parameter hash-grid model NET_1M (HashGrid 8 levels x 2^17 x 2, per-level scale 2, 2 x 32
ReLU MLP, B = 65,536) on the gauss 64^3 field for 3000 steps (model seed 5, sampler seed 6) and
requires >= 40 dB at decode, in under 600 s.  Its other arm compares against a frequency-encoded
model, an encoder outside the B200 hot path, so only the main arm is
restated here -- through the public API (build_model / InCoreSampler / train / decode / compare),
for both training engines.
"""
from __future__ import annotations

import time

import pytest

pytestmark = pytest.mark.gpu

NET_1M = {
    "encoding": {"otype": "HashGrid", "n_levels": 8, "n_features_per_level": 2,
                 "log2_hashmap_size": 17, "base_resolution": 4, "per_level_scale": 2.0},
    "network": {"n_neurons": 32, "n_hidden_layers": 2},
    "batch_size": 65536,
}


@pytest.mark.timeout(600)
@pytest.mark.parametrize("engine", [0, 1])
def test_gate3_hash_grid_convergence_main_arm(nv, engine):
    from paper_2207_11620_b200 import fields
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    from paper_2207_11620_b200.trainer import decode, train
    from paper_2207_11620_b200.volume import compare
    t0 = time.perf_counter()
    f = fields.rasterize("gauss", (64, 64, 64))
    m = build_model(NET_1M, dims=f.meta.dims, value_range=f.meta.value_range, seed=5)
    if engine == 1 and not m.tcgen05_supported():
        pytest.skip("shape outside the tcgen05 engine")
    m.train_mode = engine
    train(m, InCoreSampler(f, seed=6), steps=3000)
    q = compare(f, decode(m))
    dt = time.perf_counter() - t0
    print({"engine": engine, "n_params": m.n_params, "psnr_db": q.psnr_db, "seconds": dt})
    assert 0.9e6 <= m.n_params <= 1.3e6
    assert q.psnr_db >= 40.0, q.psnr_db
    assert dt < 600
