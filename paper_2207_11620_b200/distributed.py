"""Data-parallel training: sample sharding + the gradient exchange.

The reference is single-process; the north star adds data
parallelism by sample sharding.  Rank r of G processes the rows
[r*B/G, (r+1)*B/G) of the reference's global batch — the PCG64 stream
offset of those rows is computed exactly, so the union of the shards IS the
single-process batch — scales its loss gradient by 1/B_global
(network.py:108), and sums the flat gradient buffer plus the loss sum over the
ranks.  Two exchanges: an all-reduce followed by the identical Adam update on
every rank (parameters stay bit-identical without a broadcast), or the sharded
optimizer (the default on the device pipeline): a reduce-scatter gives rank r
the summed gradient of its 1/G slice of the flat buffer, Adam updates only that
slice (Adam time and traffic / G), and an all-gather of the updated slices
rebuilds the parameters everywhere — the same bytes on the wire as the
all-reduce.  On GPUs the collectives are NCCL over NVLink/NVSwitch captured
inside the step's CUDA graph (trainer.StepPipeline); the host logic here is
device-agnostic and is exercised with gloo on CPU in the tests.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .errors import ConfigError


def shard_rows(batch_size: int, rank: int, world: int):
    """(first row, rows) of this rank's shard of the global batch."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of world {world}")
    if batch_size % world:
        raise ConfigError(f"batch size {batch_size} is not divisible by world size {world}")
    b = batch_size // world
    return rank * b, b


def shard_u32_offset(u32_base: int, step: int, batch_size: int, row0: int) -> int:
    """u32 index of the first coordinate draw of rows [row0, ...) at `step`
    (sampler.py:54-55: each step draws 3*B float32 from the stream)."""
    return int(u32_base) + 3 * int(batch_size) * int(step) + 3 * int(row0)


def split_range(n: int, rank: int, world: int):
    """(start, count) of rank's contiguous share of n units (z-slabs / image rows);
    the first n % world ranks take one extra unit."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of world {world}")
    q, r = divmod(int(n), world)
    start = rank * q + min(rank, r)
    return start, q + (1 if rank < r else 0)


def decode_shard(model, dims=None, rank: int = 0, world: int = 1, mode: str | None = None):
    """This rank's brick of a full-grid decode (trainer.py:98-106 sharded): the
    z-slabs [z0, z0+nz) of the volume, decoded on this rank's GPU -> (z0, slab).
    Voxels are independent, so the slabs of all ranks are bit-identical to the
    single-GPU decode; the output stays distributed (no exchange)."""
    from .trainer import decode_brick
    dims = tuple(dims if dims is not None else model.dims)
    dx, dy, dz = dims
    z0, nz = split_range(dz, rank, world)
    slab = torch.empty((nz, dy, dx), dtype=torch.float32, device=model.flat_params.device)
    if nz:
        decode_brick(model, dims, z0, nz, slab, mode=mode)
    return z0, slab


def render_tile(phi, tf, cam, cfg, grid=None, rank: int = 0, world: int = 1, architecture: str = "wavefront",
                eval_mode: str | None = None):
    """This rank's image tile (rows [row0, row0+nrows)) of one ray-marched frame
    -> (row0, tile (nrows, W, 3) device tensor, FrameStats).  Rays are
    independent, so the tiles assemble bit-identically to the full frame."""
    from .render import render_frame_device
    row0, nrows = split_range(cam.height, rank, world)
    img, st = render_frame_device(phi, tf, cam, cfg, grid, architecture, eval_mode, rows=(row0, max(nrows, 1)))
    return row0, img[:nrows], st


def gather_rows(tile: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather per-rank row blocks (split_range layout) into the full (total, ...) tensor."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return tile
    world = dist.get_world_size(group)
    q = -(-total // world)
    pad = torch.zeros((q,) + tuple(tile.shape[1:]), dtype=tile.dtype, device=tile.device)
    pad[:tile.shape[0]] = tile
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][:split_range(total, r, world)[1]] for r in range(world)])


def allreduce_grads(flat_grads: torch.Tensor, loss_acc: torch.Tensor | None = None, group=None) -> None:
    """Sum the flat gradient buffer (and the loss accumulator) over ranks."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(flat_grads, op=dist.ReduceOp.SUM, group=group)
    if loss_acc is not None:
        dist.all_reduce(loss_acc, op=dist.ReduceOp.SUM, group=group)


def optimizer_shard(n: int, rank: int, world: int, align: int = 32):
    """Sharded-optimizer slice of a flat buffer of n floats: (chunk, lo, hi).
    Rank r owns [lo, hi) = [r*chunk, min(n, (r+1)*chunk)); chunk is a multiple of
    `align` floats (128 bytes), so every slice keeps the flat buffer's alignment
    modulo 128 and the float4 Adam kernel applies.  A world*chunk padded buffer
    holds the collectives' equal-sized chunks."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of world {world}")
    chunk = -(-int(n) // world)
    chunk = -(-chunk // align) * align
    lo = rank * chunk
    return chunk, lo, max(lo, min(int(n), lo + chunk))


def reduce_scatter_grads(padded_grads: torch.Tensor, out: torch.Tensor, group=None) -> None:
    """out[:chunk] = sum over ranks of padded_grads[rank*chunk:(rank+1)*chunk] (this rank's slice)."""
    world = dist.get_world_size(group)
    chunk = out.numel()
    if padded_grads.numel() != world * chunk:
        raise ConfigError("padded gradient buffer must hold world * chunk floats")
    dist.reduce_scatter_tensor(out, padded_grads, op=dist.ReduceOp.SUM, group=group)


def allgather_shards(padded: torch.Tensor, rank: int, group=None) -> None:
    """In-place all-gather: every rank's chunk of `padded` (world*chunk floats) to all ranks."""
    world = dist.get_world_size(group)
    chunk = padded.numel() // world
    dist.all_gather_into_tensor(padded, padded[rank * chunk:(rank + 1) * chunk], group=group)


def init_from_env(backend: str = "nccl"):
    """torchrun-style init (RANK / WORLD_SIZE / LOCAL_RANK / MASTER_*); returns (rank, world, local_rank)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return rank, world, local


class DataParallelTrainer:
    """Device-resident data-parallel training of one NeuralModel per rank."""

    def __init__(self, model, sampler, capacity: int, group=None, use_graph: bool = True):
        from .trainer import StepPipeline
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.pipeline = StepPipeline(model, sampler, capacity, rank=rank, world=world, group=group,
                                     use_graph=use_graph)

    def step(self, n: int = 1) -> None:
        self.pipeline.step(n)

    def finish(self):
        return self.pipeline.finish()


class PeerExchange:
    """The sharded optimizer's exchange over peer memory (NVOL_DP_PEER=1; csrc/dp_peer.cu).

    Instead of NCCL reduce-scatter -> Adam on the slice -> NCCL all-gather, every rank maps the
    other ranks' flat gradient / parameter buffers, loss sums, NaN states and step flags (CUDA IPC
    handles exchanged once through the process group; NVLink P2P between the GPUs of a node) and
    one kernel per rank (nvol_dp_fused_adam) sums its slice of all the gradients in rank order,
    updates it and writes it into every rank's parameters.  Step flags in peer memory order the
    ranks (nvol_dp_signal after the scatter, nvol_dp_wait before the next step), so the whole
    exchange lives inside the captured step graph with no collective launch.

    host_sync (NVOL_DP_PEER_HOSTSYNC=1, tests): synchronise the device and barrier the ranks
    before the fused kernel and before each step, so the flags are already set when the kernels
    read them (several ranks time-sharing ONE GPU must not spin on each other)."""

    def __init__(self, model, pipe, rank: int, world: int, group=None):
        from torch.multiprocessing.reductions import reduce_tensor
        if world > 8:
            raise ConfigError("the peer exchange supports up to 8 ranks")
        dev = model.flat_params.device
        self.rank, self.world, self.group = rank, world, group
        self.flags = torch.full((2,), int(pipe.t0), dtype=torch.int64, device=dev)
        mine = [model.flat_grads_padded, model.flat_params_padded, pipe.acc, pipe.nan_state, self.flags]
        handles = [reduce_tensor(t) for t in mine]
        everyone = [None] * world
        torch.cuda.synchronize()
        dist.all_gather_object(everyone, handles, group=group)
        self.peers = []                       # keeps the peer mappings alive
        cols = [[0] * world for _ in range(len(mine))]
        for j in range(world):
            ts = mine if j == rank else [fn(*args) for fn, args in everyone[j]]
            self.peers.append(ts)
            for a, t in enumerate(ts):
                cols[a][j] = t.data_ptr()
        from . import _lib
        self.grads, self.params, self.accs, self.nans, self.flag_ptrs = (_lib.host_i64(c) for c in cols)
        self.host_sync = os.environ.get("NVOL_DP_PEER_HOSTSYNC", "0") == "1"
        dist.barrier(group=group)

    def _sync(self) -> None:
        if self.host_sync:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def before_step(self, pipe) -> None:
        """Every rank's slices of the previous step are written; the loss sum is free."""
        from . import _lib
        self._sync()
        _lib.call("nvol_dp_wait", self.world, self.flag_ptrs, _lib.ptr(pipe.counter), _lib.ptr(pipe.acc),
                  _lib.ptr(pipe.nan_state), _lib.stream())

    def exchange_and_update(self, model, pipe) -> None:
        """After this rank's scatter: signal, then the fused reduce-scatter + Adam + all-gather."""
        from . import _lib
        _lib.call("nvol_dp_signal", _lib.ptr(self.flags), _lib.ptr(pipe.counter), _lib.ptr(pipe.nan_state),
                  _lib.stream())
        self._sync()
        _lib.call("nvol_dp_fused_adam", self.world, self.rank, self.grads, self.params, self.accs, self.nans,
                  self.flag_ptrs, pipe.slo, pipe.shi, _lib.ptr(model.flat_m), _lib.ptr(model.flat_v),
                  _lib.ptr(pipe.sched), pipe.sched.numel() // 3, _lib.ptr(pipe.counter), *pipe.adam_consts,
                  _lib.ptr(pipe.nan_state), _lib.ptr(pipe.losses), pipe.t0, pipe.capacity, 1.0 / pipe.B,
                  _lib.ptr(pipe.ticket), _lib.stream())
