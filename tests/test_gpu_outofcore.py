"""Out-of-core block buffer (sampler.py:86-297; SURVEY 8 f item 2) on the device.

Ports the reference's test_sampler.py block-buffer / out-of-core tests (their
payload oracle computed from the in-core array) and pins the sampled batches
bit-for-bit to golden vectors produced by the real reference
(oracle/gen_golden_outofcore.py).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


class ScriptedRng:
    """Replays a fixed sequence of draws (test_sampler.py:25-37)."""

    def __init__(self, steps):
        self.steps = list(steps)

    def integers(self, lo, hi, size=None):
        v = self.steps.pop(0)
        return np.full(size, v, dtype=np.int64) if size is not None else v

    def random(self, shape, dtype=np.float64):
        v = self.steps.pop(0)
        return np.full(shape, v, dtype=dtype)


def disk_volume(tmp_path, dims=(32, 20, 16), seed=5, name="vol"):
    """test_sampler.py:40-48: random float32 volume saved as sidecar + raw."""
    from paper_2207_11620_b200.volume import ScalarField, VolumeMeta, save_volume
    dx, dy, dz = dims
    data = np.random.default_rng(seed).random((dz, dy, dx)).astype(np.float32)
    f = ScalarField(VolumeMeta(dims=dims, dtype="f32", value_range=(0.0, 1.0)), data)
    side = tmp_path / f"{name}.json"
    save_volume(f, side)
    return side, data


def payload_oracle(norm, dims, origin, block_dims):
    """test_sampler.py:51-58: ghosted payload straight from the in-core array."""
    interior = [min(block_dims[a], dims[a] - origin[a]) for a in range(3)]
    gx = np.clip(np.arange(origin[0] - 1, origin[0] + interior[0] + 1), 0, dims[0] - 1)
    gy = np.clip(np.arange(origin[1] - 1, origin[1] + interior[1] + 1), 0, dims[1] - 1)
    gz = np.clip(np.arange(origin[2] - 1, origin[2] + interior[2] + 1), 0, dims[2] - 1)
    return norm[np.ix_(gz, gy, gx)], interior


def test_outofcore_matches_reference_golden(nv, tmp_path):
    """Same volume, seeds and call sequence as the reference -> identical batches,
    origins, generations and payloads."""
    from paper_2207_11620_b200.sampler import BlockBuffer, sample_outofcore
    z = golden("outofcore.npz")
    side, _ = disk_volume(tmp_path)
    buf = BlockBuffer(side, r=8, s=3, rng=np.random.default_rng(5), block_dims=(8, 8, 8))
    try:
        rng = np.random.default_rng(6)
        for k in range(4):
            b = sample_outofcore(buf, 1024, rng)
            np.testing.assert_array_equal(buf.origins, z["origins"][k])
            np.testing.assert_array_equal(b.coords.cpu().numpy(), z["coords"][k])
            np.testing.assert_array_equal(b.targets.cpu().numpy(), z["targets"][k])
            buf.refresh()
        buf.join()
        np.testing.assert_array_equal(buf.origins, z["final_origins"])
        np.testing.assert_array_equal(buf.generations, z["generations"])
        np.testing.assert_array_equal(buf.payloads.cpu().numpy(), z["payloads"])
    finally:
        buf.close()


def test_blockbuffer_initial_payloads_match_file(nv, tmp_path):
    from paper_2207_11620_b200.sampler import BlockBuffer
    side, norm = disk_volume(tmp_path)
    buf = BlockBuffer(side, r=10, s=4, rng=np.random.default_rng(7), block_dims=(8, 8, 8))
    try:
        assert np.all(buf.generations == 1)
        pay = buf.payloads.cpu().numpy()
        for slot in range(buf.r):
            origin = buf.origins[slot]
            assert np.all(origin % 8 == 0)
            want, interior = payload_oracle(norm, (32, 20, 16), origin, (8, 8, 8))
            np.testing.assert_array_equal(buf.interiors[slot], interior)
            iz, iy, ix = want.shape
            np.testing.assert_array_equal(pay[slot, :iz, :iy, :ix], want)
    finally:
        buf.close()


def test_blockbuffer_validation_and_barrier(nv, tmp_path):
    from paper_2207_11620_b200.errors import ConfigError, FormatError
    from paper_2207_11620_b200.sampler import BlockBuffer
    side, _ = disk_volume(tmp_path)
    with pytest.raises(ConfigError, match="R must be >= 1"):
        BlockBuffer(side, r=0, s=0, rng=np.random.default_rng(0))
    with pytest.raises(ConfigError, match="S must satisfy"):
        BlockBuffer(side, r=2, s=3, rng=np.random.default_rng(0), block_dims=(8, 8, 8))
    buf = BlockBuffer(side, r=4, s=2, rng=np.random.default_rng(0), block_dims=(8, 8, 8))
    try:
        buf.refresh()
        with pytest.raises(RuntimeError, match="join"):
            buf.sample(8, np.random.default_rng(0))
        buf.join()
        buf.sample(8, np.random.default_rng(0))
    finally:
        buf.close()
    raw = side.with_suffix(".raw")
    raw.write_bytes(raw.read_bytes()[:-16])
    with pytest.raises(FormatError, match="expected at least"):
        BlockBuffer(side, r=2, s=1, rng=np.random.default_rng(0), block_dims=(8, 8, 8))


def test_outofcore_zero_jitter_hits_voxel_center(nv, tmp_path):
    from paper_2207_11620_b200.sampler import BlockBuffer
    side, norm = disk_volume(tmp_path, dims=(32, 16, 16), name="pow2")
    buf = BlockBuffer(side, r=4, s=0, rng=np.random.default_rng(3), block_dims=(8, 8, 8))
    try:
        batch = buf.sample(1, ScriptedRng([2, 0.5, 0.5]))
        origin = buf.origins[2]
        voxel = np.minimum((0.5 * buf.interiors[2]).astype(np.int64), buf.interiors[2] - 1)
        center = (origin + voxel + 0.5) / np.array((32, 16, 16), dtype=np.float32)
        np.testing.assert_allclose(batch.coords.cpu().numpy()[0], center, atol=1e-7)
        gx, gy, gz = origin + voxel
        assert float(batch.targets[0]) == norm[gz, gy, gx]
        nb = buf.sample(1, ScriptedRng([2, 0.5, 0.5]), interpolation="nearest")
        assert float(nb.targets[0]) == norm[gz, gy, gx]
    finally:
        buf.close()


def test_outofcore_targets_bitwise_equal_incore(nv, tmp_path):
    """test_sampler.py:297-308: out-of-core targets == in-core trilinear of the same coords."""
    from paper_2207_11620_b200.sampler import BlockBuffer, sample_outofcore
    from paper_2207_11620_b200.volume import ScalarField, VolumeMeta, sample_trilinear_many
    side, norm = disk_volume(tmp_path)
    fld = ScalarField(VolumeMeta(dims=(32, 20, 16), dtype="f32", value_range=(0.0, 1.0)), norm)
    buf = BlockBuffer(side, r=8, s=3, rng=np.random.default_rng(5), block_dims=(8, 8, 8))
    try:
        rng = np.random.default_rng(6)
        for _ in range(4):
            batch = sample_outofcore(buf, 1024, rng)
            buf.refresh()
            want = np.clip(np.asarray(sample_trilinear_many(fld, batch.coords.cpu().numpy())), 0.0, 1.0)
            np.testing.assert_array_equal(batch.targets.cpu().numpy(), want)
    finally:
        buf.close()


def test_outofcore_sampler_trains_through_the_host_feed_pipeline(nv, tmp_path):
    """trainer.train over an OutOfCoreSampler (device batches through the H2D-fed pipeline)
    == model.train_step on the same batches."""
    from paper_2207_11620_b200 import trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import BlockBuffer, OutOfCoreSampler
    side, _ = disk_volume(tmp_path)
    cfg = {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2,
                        "log2_hashmap_size": 12, "base_resolution": 4},
           "network": {"n_neurons": 16, "n_hidden_layers": 2}, "batch_size": 2048}
    a = build_model(cfg, dims=(32, 20, 16), seed=0)
    b = build_model(cfg, dims=(32, 20, 16), seed=0)
    sa = OutOfCoreSampler(BlockBuffer(side, r=8, s=3, rng=np.random.default_rng(5), block_dims=(8, 8, 8)), seed=9)
    sb = OutOfCoreSampler(BlockBuffer(side, r=8, s=3, rng=np.random.default_rng(5), block_dims=(8, 8, 8)), seed=9)
    try:
        la = [a.train_step(sa.sample(2048)) for _ in range(4)]
        hb = trainer.train(b, sb, steps=4)
        np.testing.assert_allclose(la, hb.losses, rtol=1e-4)
        assert torch.allclose(a.flat_params, b.flat_params, atol=1e-5)
    finally:
        sa.close()
        sb.close()
