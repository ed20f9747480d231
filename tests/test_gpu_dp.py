"""Data-parallel device pipeline, two ranks sharing one GPU (gloo, eager steps): the
sharded optimizer (reduce-scatter -> slice Adam -> all-gather) and the all-reduce
exchange both reproduce the single-process trajectory of the same global batch, and
every rank ends with identical parameters and the full optimizer state."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = {"encoding": {"otype": "HashGrid", "n_levels": 8, "n_features_per_level": 2,
                    "log2_hashmap_size": 14, "base_resolution": 4},
       "network": {"n_neurons": 32, "n_hidden_layers": 2}, "batch_size": 8192}
STEPS = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dp_worker(rank, world, port, sharded, out, steps=STEPS, peer="0"):
    # NVOL_FUSED_TAIL=1 must not engage with the sharded optimizer (its step tail is the slice Adam)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NVOL_DP_SHARDED=sharded, NVOL_FUSED_TAIL="1",
                      NVOL_DP_PEER=peer, NVOL_DP_PEER_HOSTSYNC=peer)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2207_11620_b200 import fields
    from paper_2207_11620_b200.distributed import DataParallelTrainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    model = build_model(CFG, dims=(32, 32, 32), seed=0)
    fld = fields.rasterize("mlobb", (32, 32, 32))
    tr = DataParallelTrainer(model, InCoreSampler(fld, seed=1), capacity=steps, use_graph=False)
    assert tr.pipeline.sharded == (sharded == "1")
    assert not (tr.pipeline.sharded and tr.pipeline.fused)
    assert (tr.pipeline.peer is not None) == (peer == "1")
    tr.step(steps)
    losses = tr.finish()
    out[rank] = (losses, model.flat_params.cpu().numpy(), model.flat_m.cpu().numpy(), model.opt.t)
    dist.destroy_process_group()


def _run(sharded, steps=STEPS, peer="0"):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_dp_worker, args=(2, _free_port(), sharded, out, steps, peer), nprocs=2, join=True)
    return dict(out)


@pytest.mark.timeout(600)
def test_dp_two_ranks_match_single_process(nv):
    from paper_2207_11620_b200 import fields, trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    model = build_model(CFG, dims=(32, 32, 32), seed=0)
    fld = fields.rasterize("mlobb", (32, 32, 32))
    h1 = trainer.train(model, InCoreSampler(fld, seed=1), steps=1)
    one_p, one_m = model.flat_params.cpu().numpy(), model.flat_m.cpu().numpy()
    model = build_model(CFG, dims=(32, 32, 32), seed=0)
    h = trainer.train(model, InCoreSampler(fld, seed=1), steps=STEPS)
    ref_p, ref_m = model.flat_params.cpu().numpy(), model.flat_m.cpu().numpy()
    for sharded in ("1", "0"):
        # one step, tight: same global batch, gradients summed in a different order only
        # (float atomics / the exchange), so a wrong shard row offset or slice offset shows
        (l0, p0, m0, t0), (l1, p1, m1, t1) = (lambda o: (o[0], o[1]))(_run(sharded, steps=1))
        np.testing.assert_array_equal(p0, p1)
        assert l0[0] == pytest.approx(h1.losses[0], rel=1e-6)
        np.testing.assert_allclose(m0, one_m, rtol=1e-4, atol=1e-9)
        moved = np.abs(one_p - build_model(CFG, dims=(32, 32, 32), seed=0).flat_params.cpu().numpy()) > 0
        assert moved.mean() > 0.5
        # Adam's first step is ~lr * sign(g): only a gradient that cancels to ~0 (sign decided
        # by summation order) may land on the other side, by at most 2 lr
        d = np.abs(p0 - one_p)
        assert (d <= 1e-6).mean() > 0.9999 and d.max() <= 2 * 0.005 + 1e-6, (d.max(), (d > 1e-6).sum())
        out = _run(sharded)
        (l0, p0, m0, t0), (l1, p1, m1, t1) = out[0], out[1]
        np.testing.assert_array_equal(p0, p1)          # identical parameters on every rank
        np.testing.assert_array_equal(m0, m1)          # full optimizer state on every rank
        np.testing.assert_array_equal(l0, l1)
        assert t0 == t1 == STEPS
        assert l0[0] == pytest.approx(h.losses[0], rel=1e-6)   # step 0: same params, same global batch
        np.testing.assert_allclose(l0, h.losses, rtol=2e-2)
        np.testing.assert_allclose(p0, ref_p, rtol=0, atol=2e-3)
        np.testing.assert_allclose(m0, ref_m, rtol=0, atol=5e-4)


@pytest.mark.timeout(600)
def test_dp_peer_exchange_matches_single_process(nv):
    """The exchange over peer memory (NVOL_DP_PEER=1, csrc/dp_peer.cu: one kernel per rank reads its
    slice of both ranks' gradients through CUDA-IPC mappings, sums them in rank order, applies Adam
    and writes the slice into both ranks' parameters; step flags in peer memory order the ranks).
    Two ranks sharing this GPU (host-synchronised flags: NVOL_DP_PEER_HOSTSYNC=1): identical
    parameters, moments and losses on both ranks, the single-process trajectory of the same global
    batch (step 0 to 1e-6, one step's Adam update to the summation-order bound), and the same
    result as the NCCL-path sharded optimizer up to gradient summation order."""
    from paper_2207_11620_b200 import fields, trainer
    from paper_2207_11620_b200.model import build_model
    from paper_2207_11620_b200.sampler import InCoreSampler
    model = build_model(CFG, dims=(32, 32, 32), seed=0)
    fld = fields.rasterize("mlobb", (32, 32, 32))
    h1 = trainer.train(model, InCoreSampler(fld, seed=1), steps=1)
    one_p = model.flat_params.cpu().numpy()
    model = build_model(CFG, dims=(32, 32, 32), seed=0)
    h = trainer.train(model, InCoreSampler(fld, seed=1), steps=STEPS)
    (l0, p0, m0, t0), (l1, p1, m1, t1) = (lambda o: (o[0], o[1]))(_run("1", steps=1, peer="1"))
    np.testing.assert_array_equal(p0, p1)
    assert l0[0] == pytest.approx(h1.losses[0], rel=1e-6)
    d = np.abs(p0 - one_p)
    assert (d <= 1e-6).mean() > 0.9999 and d.max() <= 2 * 0.005 + 1e-6, (d.max(), (d > 1e-6).sum())
    out = _run("1", peer="1")
    (l0, p0, m0, t0), (l1, p1, m1, t1) = out[0], out[1]
    np.testing.assert_array_equal(p0, p1)
    np.testing.assert_array_equal(m0, m1)
    np.testing.assert_array_equal(l0, l1)
    assert t0 == t1 == STEPS
    assert l0[0] == pytest.approx(h.losses[0], rel=1e-6)
    np.testing.assert_allclose(l0, h.losses, rtol=2e-2)
