"""Data-parallel host logic on CPU with gloo (world_size 2).

Each rank builds its shard of the reference batch with the package's
sharding / stream-offset functions, computes its shard's gradients with the
oracle (the reference's algorithm; gradients scaled by 1/B_global), and
all-reduces them with the package's `allreduce_grads`.  The reduced
gradients and loss must equal the single-process full-batch step, and the
Adam-updated parameters must be identical on both ranks.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CFG = {"encoding": {"otype": "HashGrid", "n_levels": 4, "n_features_per_level": 2,
                    "log2_hashmap_size": 12, "base_resolution": 4},
       "network": {"n_neurons": 16, "n_hidden_layers": 2}, "batch_size": 2048}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_grads(rank, world, step):
    import nvol_oracle as orc
    from paper_2207_11620_b200.distributed import shard_rows, shard_u32_offset
    model = orc.OracleModel(CFG, seed=0)
    B = model.batch_size
    row0, b = shard_rows(B, rank, world)
    norm = orc.rasterize("mlobb", (16, 16, 16))
    coords = orc.pcg64_random_f32(1, shard_u32_offset(0, step, B, row0), 3 * b).reshape(b, 3)
    targets = orc.trilinear(norm, coords, clip=True)
    feats, idx, w = model.encode_batch(coords)
    pred, acts = orc.mlp_forward(feats, model.weights)
    diff = pred.astype(np.float64) - targets.astype(np.float64)
    dl = (np.sign(diff) / B).astype(np.float32)           # 1 / B_global (network.py:108)
    dfeat = orc.mlp_backward(acts, model.weights, model.grads, dl)
    orc.grid_encode_bwd(np.ascontiguousarray(dfeat, np.float32), idx, w, 2, model.param_grads)
    flat = np.concatenate([model.param_grads] + [g.ravel() for g in model.grads])
    return model, flat, float(np.abs(diff).sum())


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    from paper_2207_11620_b200.distributed import allreduce_grads
    model, flat, lsum = _shard_grads(rank, world, step=3)
    g = torch.from_numpy(flat.copy())
    loss = torch.tensor([lsum], dtype=torch.float64)
    allreduce_grads(g, loss)
    out[rank] = (g.numpy().copy(), float(loss.item()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_dp_gloo_matches_single_process(oracle):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    model, full, lsum = _shard_grads(0, 1, step=3)
    for r in range(world):
        g, l = out[r]
        # float sums in a different order: tolerance at fp32 rounding
        np.testing.assert_allclose(g, full, rtol=1e-5, atol=1e-9)
        assert l == pytest.approx(lsum, rel=1e-12)
    np.testing.assert_array_equal(out[0][0], out[1][0])   # identical on every rank -> identical Adam


def _sharded_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import nvol_oracle as orc
    from paper_2207_11620_b200.distributed import (allgather_shards, allreduce_grads, optimizer_shard,
                                                   reduce_scatter_grads)
    model, flat, lsum = _shard_grads(rank, world, step=3)
    n = flat.size
    p0 = np.concatenate([model.params] + [w.ravel() for w in model.weights]).astype(np.float32)
    # sharded optimizer: reduce-scatter -> Adam on this rank's slice -> all-gather
    chunk, lo, hi = optimizer_shard(n, rank, world, align=32)
    padded = torch.zeros(world * chunk)
    padded[:n] = torch.from_numpy(flat)
    gs = torch.zeros(chunk)
    reduce_scatter_grads(padded, gs)
    p = np.zeros(world * chunk, np.float32)
    p[:n] = p0
    opt = orc.AdamState()
    ps = p[lo:hi]
    orc.adam_step(opt, [ps], [gs.numpy()[:hi - lo].copy()])
    pt = torch.from_numpy(p)
    allgather_shards(pt, rank)
    # reference exchange: all-reduce + the replicated full Adam
    g = torch.from_numpy(flat.copy())
    allreduce_grads(g)
    pr = p0.copy()
    orc.adam_step(orc.AdamState(), [pr], [g.numpy().copy()])
    out[rank] = (pt.numpy()[:n].copy(), pr, opt.m[0].copy(), int(lo), int(hi))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_optimizer_gloo_equals_allreduce(oracle):
    """reduce-scatter -> slice Adam -> all-gather (the device pipeline's default
    exchange for world > 1) gives bit-identical parameters to all-reduce + the
    replicated Adam, on every rank (2 ranks, so both exchanges add the same two
    partial gradients; 18,492 floats -> 128-byte chunks with an uneven last slice)."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sharded_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        sharded, replicated, m_slice, lo, hi = out[r]
        np.testing.assert_array_equal(sharded, replicated)
        assert lo % 32 == 0 and m_slice.size == hi - lo
    np.testing.assert_array_equal(out[0][0], out[world - 1][0])


def test_optimizer_shard_layout():
    from paper_2207_11620_b200.distributed import optimizer_shard
    for n in (1, 31, 33, 18492, 12181394):
        for world in (1, 2, 3, 8):
            parts = [optimizer_shard(n, r, world) for r in range(world)]
            chunk = parts[0][0]
            assert chunk % 32 == 0 and world * chunk >= n
            spans = [(lo, hi) for _, lo, hi in parts if hi > lo]      # ranks past n own nothing
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(lo == r * chunk for r, (_, lo, hi) in enumerate(parts) if hi > lo)


def test_shard_rows_validation():
    from paper_2207_11620_b200.distributed import shard_rows
    from paper_2207_11620_b200.errors import ConfigError
    assert shard_rows(65536, 3, 8) == (24576, 8192)
    with pytest.raises(ConfigError):
        shard_rows(1000, 0, 3)
    with pytest.raises(ConfigError):
        shard_rows(1024, 2, 2)


def _gather_worker(rank, world, port, total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_11620_b200.distributed import gather_rows, split_range
    r0, n = split_range(total, rank, world)
    full = torch.arange(total * 6, dtype=torch.float32).reshape(total, 2, 3)
    got = gather_rows(full[r0:r0 + n].clone(), total)
    out[rank] = bool(torch.equal(got, full))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_tile_gather_gloo():
    """Decode bricks / render tiles: rank row blocks (split_range) reassemble exactly
    with gather_rows (uneven split: 7 rows over 3 ranks)."""
    world = 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, _free_port(), 7, out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))


def test_split_range_covers_every_unit():
    from paper_2207_11620_b200.distributed import split_range
    for n in (1, 7, 1024, 1080):
        for world in (1, 2, 3, 8):
            spans = [split_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert all(a[0] + a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert spans[-1][0] + spans[-1][1] == n
