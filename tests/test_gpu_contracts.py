"""Reference contracts the device pipeline must keep beyond the numbers:

* NaN gradients (network.py:160-183): FloatingPointError(group, flat index), the
  groups in front of the offending one updated, t not advanced, no later step
  applied -- through trainer.train (CUDA-graph pipeline), model.train_step and the
  Adam kernel itself, against the oracle's message on the same batch;
* a cached pipeline is rebuilt when anything it baked in changes (the reference
  reads opt every step);
* decode(..., to_host=True) lands the volume in host memory bit-identically
  (trainer.py:98-106 returns a host ScalarField);
* ScalarField.normalized never modifies the caller's data (volume.py:99-107);
* the out-of-core buffer never lets a queued batch read a slot that a later
  refresh overwrote (sampler.py:86-242: sampling never observes a half-written slot).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, golden_config

pytestmark = pytest.mark.gpu

CFG1 = {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2,
                     "log2_hashmap_size": 12, "base_resolution": 4},
        "network": {"n_neurons": 16, "n_hidden_layers": 2}, "batch_size": 4096}
DIMS = (32, 32, 32)


def _field(oracle):
    from paper_2207_11620_b200.volume import ScalarField, VolumeMeta
    norm = oracle.rasterize("mlobb", DIMS)
    return norm, ScalarField(VolumeMeta(DIMS, "f32", (0.0, 1.0)), norm)


@pytest.mark.parametrize("engine", [0, 1])
def test_nan_gradient_through_train_matches_reference(nv, oracle, engine):
    """A NaN parameter after 2 good steps: trainer.train raises the reference's
    FloatingPointError (same group and flat index as the oracle on the same batch),
    leaves every parameter and moment as they were before the failing step, counts
    only the applied steps in opt.t, and applies none of the steps queued behind it."""
    from paper_2207_11620_b200 import trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    if engine == 1 and not nv._lib.load().nvol_has_tcgen05(0):
        pytest.skip("no tcgen05 device")
    norm, fld = _field(oracle)
    m = build_model(CFG1, dims=DIMS, seed=0)
    m.train_mode = engine
    sampler = InCoreSampler(fld, seed=1)
    trainer.train(m, sampler, steps=2)
    ref = oracle.OracleModel(CFG1, seed=0)
    ref.load_flat(m.blob().cpu().numpy())
    bad = 3                                              # level 0 (dense): every sample reads it
    m.encoder.params[bad] = float("nan")
    ref.params[bad] = np.nan
    before = [x.clone() for x in (m.flat_params, m.flat_m, m.flat_v)]
    with pytest.raises(FloatingPointError) as got:
        trainer.train(m, sampler, steps=5)
    c, t = oracle.InCoreSampler(norm, seed=1).sample(4096 * 3)          # the reference stream ...
    c, t = c[2 * 4096:], t[2 * 4096:]                                    # ... at step 2
    ref.opt.t = 2
    with pytest.raises(FloatingPointError) as want:
        ref.train_step(c, t)
    assert str(got.value) == str(want.value)
    assert m.opt.t == 2
    for a, b in zip(before, (m.flat_params, m.flat_m, m.flat_v)):
        torch.testing.assert_close(a, b, equal_nan=True, rtol=0, atol=0)
    assert sampler.rng.u32 == 3 * 4096 * 3                               # the failing step's batch was drawn


@pytest.mark.parametrize("engine", [0, 1])
def test_nan_gradient_through_train_step_api(nv, oracle, engine):
    """model.train_step (the reference's per-call API): same error, t unchanged."""
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import SampleBatch
    if engine == 1 and not nv._lib.load().nvol_has_tcgen05(0):
        pytest.skip("no tcgen05 device")
    norm, _ = _field(oracle)
    m = build_model(CFG1, dims=DIMS, seed=0)
    m.train_mode = engine
    ref = oracle.OracleModel(CFG1, seed=0)
    c, t = oracle.InCoreSampler(norm, seed=4).sample(4096)
    t = t.copy()
    t[17] = np.nan                                        # a NaN target: that sample's gradient is NaN
    before = m.flat_params.clone()
    with pytest.raises(FloatingPointError) as got:
        m.train_step(SampleBatch(c, t, trusted=True))     # (SampleBatch's range check would reject it)
    with pytest.raises(FloatingPointError) as want:
        ref.train_step(c, t)
    assert str(got.value) == str(want.value)
    assert m.opt.t == 0
    assert torch.equal(before, m.flat_params)
    # as in the reference the un-applied gradients stay (they accumulate into the next
    # step unless zeroed); zeroed, the model trains normally again (the NaN state re-armed)
    for g in m.param_groups()[1]:
        g.zero_()
    t[17] = 0.5
    m.train_step(SampleBatch(c, t))
    assert m.opt.t == 1


def test_adam_kernel_updates_only_groups_before_the_nan(nv):
    """nvol_adam_train_step under the NaN contract: with the first NaN group's start in
    the state, exactly the groups in front of it are updated (network.py:167-171 checks
    group by group), the step is not recorded, t does not advance, the pipeline halts and
    a second launch changes nothing."""
    from paper_2207_11620_b200 import _lib
    from paper_2207_11620_b200.model import NAN_NONE, build_model
    m = build_model(golden_config(golden("encode_cfg1.npz")), dims=(8, 8, 8), seed=0)
    g = torch.randn(m.flat_size, device="cuda") * 1e-3
    starts = m.group_starts()
    gi = 2                                               # W_1
    g[starts[gi] + 5] = float("nan")
    m.flat_grads.copy_(g)
    p0 = m.flat_params.clone()
    sched = torch.tensor([0.005, 0.1, 0.001], dtype=torch.float32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    acc = torch.full((1,), 7.0, dtype=torch.float64, device="cuda")
    losses = torch.zeros(4, dtype=torch.float64, device="cuda")
    ns = torch.tensor([starts[gi], 0], dtype=torch.int64, device="cuda")
    f = lambda x: float(np.float32(x))  # noqa: E731
    args = (_lib.ptr(m.flat_params), _lib.ptr(m.flat_grads), _lib.ptr(m.flat_m), _lib.ptr(m.flat_v), m.flat_size,
            _lib.ptr(sched), 1, _lib.ptr(counter), f(0.9), f(0.1), f(0.999), f(1 - 0.999), f(1e-15), f(1e-6),
            _lib.ptr(ns), _lib.ptr(acc), _lib.ptr(losses), 0, 4, 1.0, _lib.ptr(ticket), _lib.stream())
    _lib.call("nvol_adam_train_step", *args)
    p1 = m.flat_params.clone()
    assert not torch.equal(p1[:starts[gi]], p0[:starts[gi]])          # groups 0, 1 updated
    assert torch.equal(p1[starts[gi]:], p0[starts[gi]:])              # W_1 and later untouched
    assert torch.equal(m.flat_grads[starts[gi]:].nan_to_num(), g[starts[gi]:].nan_to_num())   # not consumed
    assert not m.flat_grads[:starts[gi]].abs().sum().item()           # consumed gradients zeroed
    assert int(counter.item()) == 0 and float(acc.item()) == 7.0 and not losses.abs().sum().item()
    assert ns.tolist() == [starts[gi], 1]                             # halted
    _lib.call("nvol_adam_train_step", *args)
    assert torch.equal(m.flat_params, p1)
    assert int(counter.item()) == 0
    # a clean state advances as usual
    ns.copy_(torch.tensor([NAN_NONE, 0]))
    m.flat_grads.zero_()
    _lib.call("nvol_adam_train_step", *args)
    assert int(counter.item()) == 1 and float(losses[0].item()) == 7.0


def test_cached_pipeline_rebuilt_when_optimizer_changes(nv, oracle):
    """Changing opt (lr, betas, l2) or the loss between train() calls takes effect:
    the pipeline that baked the old values into its graphs is not reused."""
    from paper_2207_11620_b200 import trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    _, fld = _field(oracle)
    m = build_model(CFG1, dims=DIMS, seed=0)
    s = InCoreSampler(fld, seed=1)
    trainer.train(m, s, steps=3)
    p = m._pipeline
    trainer.train(m, s, steps=2)
    assert m._pipeline is p                                           # unchanged: reused
    m.opt.base_lr = 0.0
    m.opt.l2_reg = 0.0
    trainer.train(m, s, steps=2)
    assert m._pipeline is not p
    before = m.flat_params.clone()
    trainer.train(m, s, steps=2)                                      # lr 0, no l2: Adam moves nothing
    assert torch.equal(before, m.flat_params)
    m.loss_kind = "L2"
    q = m._pipeline
    trainer.train(m, s, steps=1)
    assert m._pipeline is not q


def test_decode_to_host_is_bit_identical(nv, monkeypatch):
    """decode(to_host=True) (ring of device slabs, overlapped D2H) == the device decode,
    with several slabs in flight and a ragged last slab."""
    from paper_2207_11620_b200 import trainer
    from paper_2207_11620_b200.model import build_model
    m = build_model(golden_config(golden("encode_cfg2.npz")), dims=(40, 24, 37), seed=0)
    r = np.random.default_rng(2)
    m.encoder.params.copy_(torch.from_numpy(r.normal(0, 0.3, m.encoder.params.shape).astype(np.float32)))
    dev = trainer.decode(m).data.cpu().numpy()
    monkeypatch.setattr(trainer, "_HOST_SLAB_BYTES", 40 * 24 * 4 * 5)      # 5-row slabs: 8 slabs, ragged
    host = trainer.decode(m, to_host=True)
    assert isinstance(host.data, np.ndarray) and host.data.dtype == np.float32
    np.testing.assert_array_equal(host.data, dev)
    np.testing.assert_array_equal(trainer.decode(m, slab_z=3, to_host=True).data, dev)


def test_normalized_does_not_modify_data(nv):
    from paper_2207_11620_b200.volume import ScalarField, VolumeMeta, mse
    d = torch.tensor(np.linspace(-0.5, 1.5, 4 * 4 * 4, dtype=np.float32).reshape(4, 4, 4)).cuda()
    keep = d.clone()
    f = ScalarField(VolumeMeta((4, 4, 4), "f32", (0.0, 1.0)), d)
    n = f.normalized
    assert torch.equal(d, keep)
    assert float(n.min()) == 0.0 and float(n.max()) == 1.0
    # u8 data: the reference normalises in float64 (normalized_as(np.float64))
    a = np.random.default_rng(0).integers(0, 256, (8, 8, 8)).astype(np.uint8)
    b = np.random.default_rng(1).integers(0, 256, (8, 8, 8)).astype(np.uint8)
    fa = ScalarField(VolumeMeta((8, 8, 8), "u8", (3.0, 250.0)), a)
    fb = ScalarField(VolumeMeta((8, 8, 8), "u8", (3.0, 250.0)), b)
    na = np.clip((a.astype(np.float64) - 3.0) / 247.0, 0, 1)
    nb = np.clip((b.astype(np.float64) - 3.0) / 247.0, 0, 1)
    assert mse(fa, fb) == pytest.approx(float(np.mean((na - nb) ** 2)), rel=1e-14)


def test_outofcore_refresh_never_races_queued_batches(nv, tmp_path):
    """Many host-run-ahead steps with a tiny buffer (R = 2, S = 2: every slot is
    replaced after every batch): each batch's targets equal the in-core trilinear of
    its coordinates, i.e. no queued sampling launch ever read a slot or origin table
    that a later refresh had already overwritten."""
    from paper_2207_11620_b200.sampler import BlockBuffer, OutOfCoreSampler
    from paper_2207_11620_b200.volume import ScalarField, VolumeMeta, save_volume
    import nvol_oracle as orc
    dims = (48, 40, 36)
    data = np.random.default_rng(9).random((dims[2], dims[1], dims[0])).astype(np.float32)
    side = tmp_path / "v.json"
    save_volume(ScalarField(VolumeMeta(dims=dims, dtype="f32", value_range=(0.0, 1.0)), data), side)
    buf = BlockBuffer(side, r=2, s=2, rng=np.random.default_rng(3), block_dims=(16, 16, 16))
    s = OutOfCoreSampler(buf, seed=4)
    batches = []
    try:
        torch.cuda._sleep(50_000_000)            # keep the device busy so the host runs far ahead
        for _ in range(40):
            batches.append(s.sample(2048))
        torch.cuda.synchronize()
        for bt in batches:
            c = bt.coords.cpu().numpy()
            np.testing.assert_array_equal(bt.targets.cpu().numpy(), orc.trilinear(data, c, clip=True))
    finally:
        s.close()


def test_vnr_written_by_the_reference_loads_and_round_trips(nv, tmp_path):
    """a .vnr the reference wrote (oracle/gen_golden_vnr.py, trainer.py:125-138)
    loads here with its config, dims and value range; eval_fused is bit-identical to the
    reference's; decode matches the reference's decode (eval_batch, BLAS-ordered, so to
    float rounding); and save_model writes the reference's file back byte for byte."""
    from conftest import GOLDEN
    from paper_2207_11620_b200 import trainer
    z = golden("vnr_cfg1.npz")
    m = trainer.load_model(GOLDEN / "ref_cfg1.vnr")
    assert m.dims == (48, 48, 48) and tuple(m.value_range) == (2.0, 5.0)
    np.testing.assert_array_equal(m.eval_fused(z["coords"]), z["eval_fused"])
    np.testing.assert_allclose(m.eval_batch(z["coords"]), z["eval_batch"], rtol=0, atol=1e-6)
    d = trainer.decode(m, dims=tuple(int(x) for x in z["dims"]), to_host=True).data
    np.testing.assert_allclose(d, z["decode"], rtol=0, atol=3e-6 * 3.0)
    out = tmp_path / "again.vnr"
    trainer.save_model(m, out)
    assert out.read_bytes() == (GOLDEN / "ref_cfg1.vnr").read_bytes()
