"""Training orchestration, decoding and model serialisation on the B200.

Mirror of the reference's trainer.py (/root/reference/pkg/src/neuralvol/
trainer.py): TrainHistory, train, decode_slabs, decode, compression_ratio,
save_model / load_model with the byte-identical "VNRM" v1 format.

`train` with a device InCoreSampler and a float32 grid model runs the
device-resident pipeline (StepPipeline): per step one sampling kernel, the
fused forward/backward, one flat Adam kernel and a device-side loss record,
captured once into a CUDA graph and replayed — no host round trip per step.
The per-step losses are read back once at the end.
"""
from __future__ import annotations

import csv
import gc
import json
import logging
import struct
import os
import time
import weakref
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, FormatError
from .model import MODE_TCGEN05, NAN_NONE, TRAIN_ENCODE_ONLY, TRAIN_PREENCODED, NeuralModel, build_model
from .network import adam_scalars, lr_at
from .sampler import InCoreSampler
from .volume import ScalarField, VolumeMeta

log = logging.getLogger(__name__)

MODEL_MAGIC = b"VNRM"
MODEL_VERSION = 1


@dataclass
class TrainHistory:
    """trainer.py:30-58."""
    steps: list = field(default_factory=list)
    losses: list = field(default_factory=list)
    lrs: list = field(default_factory=list)
    wall_ms: list = field(default_factory=list)

    def append(self, step: int, loss: float, lr: float, ms: float) -> None:
        if self.steps and step <= self.steps[-1]:
            raise ConfigError(f"history steps must increase: {step} after {self.steps[-1]}")
        self.steps.append(step)
        self.losses.append(loss)
        self.lrs.append(lr)
        self.wall_ms.append(ms)

    def to_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["step", "loss", "lr", "ms"])
            for row in zip(self.steps, self.losses, self.lrs, self.wall_ms):
                w.writerow([row[0], f"{row[1]:.8g}", f"{row[2]:.8g}", f"{row[3]:.3f}"])

    @staticmethod
    def from_csv(path) -> "TrainHistory":
        h = TrainHistory()
        with open(path, newline="") as fh:
            for row in csv.DictReader(fh):
                h.append(int(row["step"]), float(row["loss"]), float(row["lr"]), float(row["ms"]))
        return h


class StepPipeline:
    """Device-resident training steps (model.py:154-174 + sampler.py:263-270 + network.py:160-183).

    One step = fused forward/backward of the batch sampled for it (rows
    [row0, row0+b) of the global batch) -> [all-reduce of the flat gradient +
    loss, when data-parallel] -> Adam + loss record + step-counter advance
    (one kernel).  The NEXT step's batch is sampled on a side stream while
    this step's encode / MLP / scatter run (double-buffered coordinates), so
    sampling leaves the critical path.  Everything reads the device step
    counter, so two captured CUDA graphs (even / odd buffer parity) replay
    every step."""

    def __init__(self, model: NeuralModel, sampler: InCoreSampler, capacity: int, rank: int = 0, world: int = 1,
                 group=None, use_graph: bool = True, mc_grid=None):
        if not model._use_kernels():
            raise ConfigError("the device pipeline needs a float32 grid model")
        from .distributed import shard_rows
        B = model.batch_size
        row0, b = shard_rows(B, rank, world)
        # weak: the model caches its pipeline (model._pipeline), and a strong cycle would
        # leave the old pipeline's graphs / streams / events to the cyclic collector,
        # which can run inside a later graph capture and invalidate it
        self._model = weakref.ref(model)
        self.sampler = sampler
        self.train_mode = model._engine()
        self.B, self.b, self.row0 = B, b, row0
        self.rank = rank
        self.world, self.group = world, group
        # sharded optimizer (distributed.py): reduce-scatter -> Adam on this rank's slice ->
        # all-gather; NVOL_DP_SHARDED=0 restores all-reduce + replicated Adam
        self.sharded = world > 1 and os.environ.get("NVOL_DP_SHARDED", "1") != "0"
        if self.sharded:
            from .distributed import optimizer_shard
            self.chunk, self.slo, self.shi = optimizer_shard(model.flat_size, rank, world)
            if getattr(model, "flat_params_padded", None) is None or model.flat_params_padded.numel() != world * self.chunk:
                model.rehome_flat(world * self.chunk)
            self.gslice = torch.zeros(model.flat_lead + self.chunk, dtype=torch.float32,
                                      device=model.flat_params.device)[model.flat_lead:]
        dev = model.flat_params.device
        self.bufs = [(torch.empty((self.b, 3), dtype=torch.float32, device=dev),
                      torch.empty(self.b, dtype=torch.float32, device=dev)) for _ in range(2)]
        self.coords, self.targets = self.bufs[0]
        self.t0 = model.opt.t
        self.counter = torch.full((1,), self.t0, dtype=torch.int64, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        # host feed: any sampler yielding host batches (sampler.py:263-297 protocol);
        # each step's batch is DMA'd from pinned memory on a copy stream while the
        # previous step computes, and each step's loss is read back asynchronously
        self.host_feed = not isinstance(sampler, InCoreSampler)
        self.u32_base = 0 if self.host_feed else sampler.rng.u32
        self.capacity = int(capacity)
        self.losses = torch.zeros(self.capacity, dtype=torch.float64, device=dev)
        self.acc = torch.zeros(1, dtype=torch.float64, device=dev)
        # NaN contract (nvol.h): [first NaN group's flat start, halted]; checked by every step kernel
        self.nan_state = torch.tensor([NAN_NONE, 0], dtype=torch.int64, device=dev)
        o = model.opt
        rows = []
        for t in range(self.t0 + self.capacity + 1):
            lr, c1, c2 = adam_scalars(o, t)
            rows.append((lr, c1, c2))
        self.sched = torch.tensor(np.asarray(rows, dtype=np.float64).astype(np.float32), device=dev).reshape(-1)
        f = lambda x: float(np.float32(x))  # noqa: E731  dt(...) of network.py:172-181
        self.adam_consts = (f(o.beta1), f(1.0 - o.beta1), f(o.beta2), f(1.0 - o.beta2), f(o.epsilon), f(o.l2_reg))
        # Optional L2 set-aside for persisting lines (NVOL_L2_PERSIST bytes).  Off by
        # default: measured on B200 it starves Adam's streaming (step 189 -> 267 us).
        persist = int(os.environ.get("NVOL_L2_PERSIST", "0"))
        self.l2_persist = int(_lib.load().nvol_l2_persist(persist)) if persist > 0 else 0
        # online macro-cells (OnlineMacrocells tap): fused into the sampler kernel /
        # applied to the staged host batch; sampling stays in step (no look-ahead)
        # so the grid sees exactly the trained batches
        self.mc_grid = mc_grid
        self.overlap = ((not self.host_feed) and mc_grid is None
                        and os.environ.get("NVOL_SAMPLE_OVERLAP", "1") != "0")
        self.side = torch.cuda.Stream(device=dev) if self.overlap else None
        # fused step tail (opt-in, NVOL_FUSED_TAIL=1): Adam + the NEXT batch's encoder
        # forward in one launch (nvol_adam_encode_step); the next step's fwd/bwd then
        # skips its encode.  Off by default: measured on B200 at cfg2 the two halves
        # share L2 throughput, so the fused launch (145 us) is slower than Adam +
        # encode back to back (70 + 31 us) -- DESIGN.md "Step-tail fusion"
        # (not with the sharded optimizer: its step tail is the slice Adam + all-gather)
        self.fused = (self.overlap and self.train_mode == MODE_TCGEN05 and not self.sharded
                      and os.environ.get("NVOL_FUSED_TAIL", "0") == "1")
        # the tcgen05 engine records a fork event after its encode launch (NVOL_FORK_AFTER_ENCODE=0:
        # fork at the start of the step)
        self.fork_after_encode = (self.overlap and not self.fused and model._engine() == MODE_TCGEN05
                                  and model._tc_device() and os.environ.get("NVOL_FORK_AFTER_ENCODE", "1") != "0")
        self.fork_ev = torch.cuda.Event() if self.fork_after_encode else None
        self.fingerprint = pipeline_fingerprint(model)
        # the sharded exchange over peer memory instead of NCCL (NVOL_DP_PEER=1, distributed.PeerExchange)
        self.peer = None
        if self.sharded and os.environ.get("NVOL_DP_PEER", "0") == "1":
            from .distributed import PeerExchange
            self.peer = PeerExchange(model, self, rank, world, group)
        self.work = torch.zeros(2 + 32, dtype=torch.int32, device=dev)   # NVOL_MAX_LEVELS
        if self.host_feed:
            self.copy_stream = torch.cuda.Stream(device=dev)
            self.ready = [torch.cuda.Event(), torch.cuda.Event()]
            self.free = [torch.cuda.Event(), torch.cuda.Event()]
            self.staged = [None, None]          # host tensors whose DMA may still be in flight
            self.staging = [None, None]         # pinned staging for non-pinned host batches
            self.loss_host = torch.zeros(self.capacity, dtype=torch.float64).pin_memory()
            # each step's loss is read back on its own stream (after the step's event), so the
            # 8-byte D2H never sits between two steps on the main stream
            self.d2h_stream = torch.cuda.Stream(device=dev)
        self.use_graph = use_graph
        self.graphs = [None, None]
        self.done = 0

    @property
    def model(self) -> NeuralModel:
        m = self._model()
        if m is None:
            raise ConfigError("the pipeline's model was released")
        return m

    def sample_into(self, parity: int, ahead: int) -> None:
        """Sample the batch of step (device counter + ahead) into buffer `parity`."""
        s = self.sampler
        vol = s.volume
        dz, dy, dx = vol.shape
        c, t = self.bufs[parity]
        # the kernel offsets by (counter - counter0): counter0 = t0 - ahead
        g = self.mc_grid
        gx, gy, gz = g.grid_dims if g is not None else (0, 0, 0)
        _lib.call("nvol_sample_incore_dev_mc", *s.rng.words(), self.u32_base, _lib.ptr(self.counter),
                  self.t0 - ahead, self.B, self.row0, self.b, _lib.ptr(vol), dx, dy, dz, _lib.ptr(c), _lib.ptr(t),
                  _lib.ptr(g.value_lo) if g is not None else None, _lib.ptr(g.value_hi) if g is not None else None,
                  gx, gy, gz, g.n_g if g is not None else 1, _lib.stream())

    def _feed(self, parity: int) -> None:
        """H2D of this step's host batch into device buffer `parity` (copy stream)."""
        batch = self.sampler.sample(self.B)
        if len(batch) != self.B:
            raise ConfigError(f"batch size {len(batch)} != configured {self.B}")
        hc, ht = batch.coords, batch.targets
        r0, r1 = self.row0, self.row0 + self.b
        on_device = isinstance(hc, torch.Tensor) and hc.is_cuda
        if on_device:
            hc = hc.to(torch.float32)[r0:r1]
            ht = ht.to(torch.float32)[r0:r1]
            self.copy_stream.wait_stream(torch.cuda.current_stream())
        elif not (isinstance(hc, torch.Tensor) and hc.is_pinned() and hc.dtype == torch.float32
                  and isinstance(ht, torch.Tensor) and ht.is_pinned() and ht.dtype == torch.float32):
            if self.staging[parity] is None:
                self.staging[parity] = (torch.empty((self.b, 3), dtype=torch.float32).pin_memory(),
                                        torch.empty(self.b, dtype=torch.float32).pin_memory())
            self.ready[parity].synchronize()    # the staging buffer's previous DMA is done
            sc, st = self.staging[parity]
            sc.numpy()[...] = np.asarray(hc[r0:r1], dtype=np.float32)
            st.numpy()[...] = np.asarray(ht[r0:r1], dtype=np.float32)
            hc, ht = sc, st
        elif not on_device:
            hc, ht = hc[r0:r1], ht[r0:r1]
        c, t = self.bufs[parity]
        self.copy_stream.wait_event(self.free[parity])   # the step that last read this buffer is done
        with torch.cuda.stream(self.copy_stream):
            c.copy_(hc, non_blocking=True)
            t.copy_(ht, non_blocking=True)
        self.ready[parity].record(self.copy_stream)
        self.staged[parity] = (hc, ht)
        torch.cuda.current_stream().wait_event(self.ready[parity])

    def _body(self, parity: int) -> None:
        m = self.model
        main = torch.cuda.current_stream()
        if self.peer is not None:
            self.peer.before_step(self)
        if self.host_feed:
            if self.mc_grid is not None:
                from .macrocell import macrocell_update_online
                from .sampler import SampleBatch
                macrocell_update_online(self.mc_grid, SampleBatch(*self.bufs[parity], trusted=True))
        elif self.overlap:
            self.side.wait_stream(main)                 # fork: next step's batch on the side stream
            if not self.fork_after_encode:
                with torch.cuda.stream(self.side):
                    self.sample_into(parity ^ 1, 1)
        else:
            self.sample_into(parity, 0)
        c, t = self.bufs[parity]
        if self.fork_after_encode:
            # fork the next step's sampling after this step's encode (nvol_set_fork_event): the
            # sampler then overlaps the latency-bound MLP, not the L2-bound encoder
            _lib.call("nvol_set_fork_event", self.fork_ev.cuda_event)
            try:
                m.fwd_bwd_device(c, t, self.acc, b_global=self.B, nan_state=self.nan_state)
            finally:
                _lib.call("nvol_set_fork_event", None)
            self.side.wait_event(self.fork_ev)
            with torch.cuda.stream(self.side):
                self.sample_into(parity ^ 1, 1)
        else:
            m.fwd_bwd_device(c, t, self.acc, b_global=self.B, flags=TRAIN_PREENCODED if self.fused else 0,
                             nan_state=self.nan_state)
        if self.peer is not None:
            if self.overlap:
                main.wait_stream(self.side)
            self.peer.exchange_and_update(m, self)
            return
        if self.sharded:
            import torch.distributed as dist
            from .distributed import allgather_shards, reduce_scatter_grads
            reduce_scatter_grads(m.flat_grads_padded, self.gslice, self.group)
            dist.all_reduce(self.acc, group=self.group)
            dist.all_reduce(self.nan_state[:1], op=dist.ReduceOp.MIN, group=self.group)
            m.flat_grads_padded.zero_()                 # this rank's gradient is consumed
            if self.overlap:
                main.wait_stream(self.side)
            o4 = 4 * self.slo
            _lib.call("nvol_adam_train_step", _lib.ptr(m.flat_params) + o4, _lib.ptr(self.gslice),
                      _lib.ptr(m.flat_m) + o4, _lib.ptr(m.flat_v) + o4, self.shi - self.slo, _lib.ptr(self.sched),
                      self.sched.numel() // 3, _lib.ptr(self.counter), *self.adam_consts, _lib.ptr(self.nan_state),
                      _lib.ptr(self.acc), _lib.ptr(self.losses), self.t0, self.capacity, 1.0 / self.B,
                      _lib.ptr(self.ticket), _lib.stream())
            allgather_shards(m.flat_params_padded, self.rank, self.group)
            return
        if self.world > 1:
            from .distributed import allreduce_grads
            allreduce_grads(m.flat_grads, self.acc, self.group)
            import torch.distributed as dist
            dist.all_reduce(self.nan_state[:1], op=dist.ReduceOp.MIN, group=self.group)
        if self.overlap:
            main.wait_stream(self.side)                 # join before the counter advances
        if self.fused:
            cfg = m.encoder.config
            off, res, ent, dense = m.encoder.c_tables()
            ws = m._workspace(self.b)
            _lib.call("nvol_adam_encode_step", _lib.ptr(m.flat_params), _lib.ptr(m.flat_grads), _lib.ptr(m.flat_m),
                      _lib.ptr(m.flat_v), m.flat_size, _lib.ptr(self.sched), self.sched.numel() // 3,
                      _lib.ptr(self.counter), *self.adam_consts, _lib.ptr(self.nan_state), _lib.ptr(self.acc),
                      _lib.ptr(self.losses), self.t0, self.capacity, 1.0 / self.B, _lib.ptr(self.work),
                      _lib.ptr(self.bufs[parity ^ 1][0]), self.b, off, res, ent, dense, cfg.n_levels,
                      cfg.n_features_per_level, m.mlp.config.n_neurons, m.mlp.config.n_hidden_layers,
                      _lib.ptr(ws), ws.numel(), _lib.stream())
            return
        _lib.call("nvol_adam_train_step", _lib.ptr(m.flat_params), _lib.ptr(m.flat_grads), _lib.ptr(m.flat_m),
                  _lib.ptr(m.flat_v), m.flat_size, _lib.ptr(self.sched), self.sched.numel() // 3,
                  _lib.ptr(self.counter), *self.adam_consts, _lib.ptr(self.nan_state), _lib.ptr(self.acc),
                  _lib.ptr(self.losses), self.t0, self.capacity, 1.0 / self.B, _lib.ptr(self.ticket), _lib.stream())

    def launches_per_step(self) -> int:
        """Kernels of one step from this library (for the bench's gpu_launches)."""
        if self.train_mode == 0:
            return 1 + 5 + 3 * (self.model.mlp.config.n_hidden_layers + 1) + 1 + 1
        pack = 0 if os.environ.get("NVOL_MLP4", "1") == "0" else 1
        if self.fused:
            # sample (next step's), the weight image, MLP, the dW fold, scatter, Adam + next encode
            fold = 1 if (pack and os.environ.get("NVOL_DW_PARTIALS", "1") != "0") else 0
            return 1 + pack + 2 + fold + 1
        # sample (next step's, overlapped), the MLP weight image (pack_w4, side stream; four-slot
        # MLP kernel), nchunks x (encode, MLP, scatter), the dW fold, Adam step
        # (chunk plan of train_tc.cu make_plan: NVOL_TRAIN_CHUNKS, default 1)
        ntiles = (self.b + 127) // 128
        nc = max(1, min(int(os.environ.get("NVOL_TRAIN_CHUNKS", "1")), 4, ntiles))
        ct = (ntiles + nc - 1) // nc
        nc = (ntiles + ct - 1) // ct
        # the MLP's dW partials folded beside the scatter (dw_reduce_kernel; one MLP launch only)
        fold = 1 if (pack and nc == 1 and os.environ.get("NVOL_DW_PARTIALS", "1") != "0") else 0
        return 1 + pack + 3 * nc + fold + 1

    def step(self, n: int = 1) -> None:
        """Enqueue n steps (no host synchronisation)."""
        if self.done + n > self.capacity:
            raise ConfigError(f"pipeline capacity {self.capacity} exceeded")
        for k in range(n):
            parity = self.done & 1
            if self.host_feed:
                self._feed(parity)
            if self.done == 0 and self.overlap:
                self.sample_into(0, 0)                  # the first batch, on the main stream
            if k == 0 and self.fused:
                # this call's first batch: encode it with the current parameters (the
                # previous call's look-ahead encode may predate a parameter change)
                c, t = self.bufs[parity]
                self.model.fwd_bwd_device(c, t, self.acc, b_global=self.B, flags=TRAIN_ENCODE_ONLY,
                                          nan_state=self.nan_state)
            if self.done == 0:
                self._body(parity)                      # eager first step (warms up / lazily allocates)
            elif not self.use_graph:
                self._body(parity)
            else:
                if self.graphs[parity] is None:
                    g = torch.cuda.CUDAGraph()
                    # no cyclic collection mid-capture: a destructor's CUDA call (event /
                    # stream / graph teardown) would invalidate the capture
                    gc_was = gc.isenabled()
                    gc.disable()
                    try:
                        with torch.cuda.graph(g):
                            self._body(parity)
                    finally:
                        if gc_was:
                            gc.enable()
                    self.graphs[parity] = g
                self.graphs[parity].replay()
            if self.host_feed:
                main = torch.cuda.current_stream()
                self.free[parity].record(main)
                self.d2h_stream.wait_event(self.free[parity])
                with torch.cuda.stream(self.d2h_stream):
                    self.loss_host[self.done:self.done + 1].copy_(self.losses[self.done:self.done + 1],
                                                                  non_blocking=True)
            self.done += 1

    def finish(self) -> np.ndarray:
        """Synchronise, commit host-side state, return the per-step losses.

        NaN contract (network.py:160-183): a step whose gradient holds a NaN updated only
        the parameter groups in front of the offending one and halted the pipeline; the
        steps queued after it did nothing.  opt.t counts the applied steps only, the
        sampler stands after the failing step's batch (drawn, as the reference draws it
        before train_step raises), and FloatingPointError(group, flat index) is raised."""
        m = self.model
        if self.host_feed:
            torch.cuda.current_stream().synchronize()
            self.d2h_stream.synchronize()
            losses = self.loss_host[:self.done].numpy().copy()
            self.staged = [None, None]
        else:
            losses = self.losses[:self.done].cpu().numpy()
        if self.sharded:
            # every rank holds the whole optimizer state again
            from .distributed import allgather_shards
            allgather_shards(m.flat_m_padded, self.rank, self.group)
            allgather_shards(m.flat_v_padded, self.rank, self.group)
        lim = int(self.nan_state[0].item())
        applied = self.done if lim == NAN_NONE else int(self.counter.item()) - self.t0
        m.opt.t = self.t0 + applied
        if not self.host_feed:
            self.sampler.rng.u32 = self.u32_base + 3 * self.B * (applied + (lim != NAN_NONE))
        if lim == NAN_NONE:
            return losses
        if self.sharded:
            # the summed gradient of the failing step lives in the ranks' slices
            from .distributed import allgather_shards
            n = self.shi - self.slo
            m.flat_grads_padded[self.rank * self.chunk:self.rank * self.chunk + n].copy_(self.gslice[:n])
            allgather_shards(m.flat_grads_padded, self.rank, self.group)
        err = m.nan_error(lim)
        m._pipeline = None                      # halted: the next train() builds a fresh pipeline
        raise err


def pipeline_fingerprint(model: NeuralModel) -> tuple:
    """Everything a StepPipeline bakes in at construction (Adam schedule and constants,
    loss / output activation captured in its graphs, engine, batch, buffers): a cached
    pipeline is reused only while this is unchanged (the reference reads opt every step)."""
    o = model.opt
    return (o.base_lr, o.beta1, o.beta2, o.epsilon, o.l2_reg, o.decay_start, o.decay_interval, o.decay_base,
            model.loss_kind, model.mlp.config.output_activation, model._engine(), model.batch_size,
            model.flat_params.data_ptr())


def _cached_pipeline(model: NeuralModel, sampler, steps: int, mc_grid=None) -> "StepPipeline":
    """Reuse the model's pipeline (and its captured graphs) across train() calls
    while nothing it baked in changed: same sampler object, optimizer step and
    (device sampling) stream position, and capacity left."""
    p = getattr(model, "_pipeline", None)
    if p is not None:
        ok = (p.sampler is sampler and p.mc_grid is mc_grid and p.t0 + p.done == model.opt.t
              and p.done + steps <= p.capacity
              and p.fingerprint == pipeline_fingerprint(model)
              and (p.host_feed or sampler.rng.u32 == p.u32_base + 3 * p.B * p.done))
        if ok:
            return p
    p = StepPipeline(model, sampler, max(steps, 256), mc_grid=mc_grid)
    model._pipeline = p
    return p


def _fast_path(model, sampler, tap) -> bool:
    from .macrocell import OnlineMacrocells
    if (tap is not None and not isinstance(tap, OnlineMacrocells)) or not model._use_kernels():
        return False
    if isinstance(sampler, InCoreSampler):
        return sampler.interpolation == "trilinear"
    return os.environ.get("NVOL_HOST_FEED", "1") != "0"   # host batches: the H2D-overlapped pipeline


def train(model: NeuralModel, sampler, steps: int, tap=None, log_every: int = 0) -> TrainHistory:
    """Run `steps` optimisation steps, drawing one batch per step (trainer.py:61-77)."""
    if steps < 1:
        raise ConfigError(f"steps must be >= 1, got {steps}")
    history = TrainHistory()
    if _fast_path(model, sampler, tap):
        t0 = model.opt.t
        pipe = _cached_pipeline(model, sampler, steps, mc_grid=tap.grid if tap is not None else None)
        start = time.perf_counter()
        first = pipe.done
        pipe.step(steps)
        losses = pipe.finish()[first:]
        ms = (time.perf_counter() - start) * 1e3 / steps
        for k in range(steps):
            history.append(t0 + k, float(losses[k]), lr_at(model.opt, t0 + k), ms)
            if log_every and (t0 + k + 1) % log_every == 0:
                log.info("step %d  loss %.6f  lr %.5g", t0 + k + 1, losses[k], history.lrs[-1])
        return history
    for _ in range(steps):
        t0 = time.perf_counter()
        step_index = model.opt.t
        batch = sampler.sample(model.batch_size)
        loss = model.train_step(batch)
        if tap is not None:
            tap(batch)
        ms = (time.perf_counter() - t0) * 1e3
        history.append(step_index, loss, lr_at(model.opt, step_index), ms)
        if log_every and (step_index + 1) % log_every == 0:
            log.info("step %d  loss %.6f  lr %.5g  %.1f ms", step_index + 1, loss, history.lrs[-1], ms)
    return history


def decode_brick(model: NeuralModel, dims, z0: int, nz: int, out: torch.Tensor, mode: str | None = None) -> None:
    """Voxel-centre decode of rows [z0, z0+nz) into out (device, nz*dy*dx f32)."""
    dx, dy, dz = dims
    lo, hi = model.value_range
    c = model.encoder.config
    off, res, ent, dense = model.encoder.c_tables()
    widths = model._widths()
    mode = mode or model.infer_mode
    _lib.call("nvol_decode", _lib.ptr(model.flat_params), off, res, ent, dense, c.n_levels, c.n_features_per_level,
              _lib.ptr(model._weights_flat()), _lib.host_i32(widths), len(widths) - 1,
              int(model.mlp.config.output_activation == "relu"), dx, dy, dz, z0, nz, float(lo), float(hi),
              _lib.ptr(out), {"exact": 0, "tensor": 1, "centres64": 2}[mode],
              _lib.ptr(model.mlp_image()) if mode == "tensor" else None, _lib.stream())


def decode_slabs(model: NeuralModel, dims=None, slab_z: int = 16):
    """Yield (z0, slab) of the decoded volume in ascending z (trainer.py:80-95); slabs are device tensors."""
    if slab_z < 1:
        raise ConfigError("slab_z must be >= 1")
    dims = tuple(dims if dims is not None else model.dims)
    dx, dy, dz = dims
    _require_grid_model(model)
    for z0 in range(0, dz, slab_z):
        nz = min(slab_z, dz - z0)
        slab = torch.empty((nz, dy, dx), dtype=torch.float32, device=model.flat_params.device)
        decode_brick(model, dims, z0, nz, slab)
        yield z0, slab


def _require_grid_model(model) -> None:
    if not model._use_kernels():
        raise ConfigError("decode runs on float32 grid models")


def decode(model: NeuralModel, dims=None, slab_z: int | None = None, to_host: bool = False) -> ScalarField:
    """Evaluate Phi at every voxel centre and denormalise by value_range (trainer.py:98-106).

    The whole volume is decoded by one launch (slab boundaries cannot change
    any value: each voxel is evaluated independently); slab_z only chunks the
    launches.  The result stays on the device unless to_host, which lands it in
    host memory as the reference does (a numpy f32 array), with each slab's D2H
    overlapped with the next slab's decode (_decode_to_host)."""
    dims = tuple(dims if dims is not None else model.dims)
    dx, dy, dz = dims
    _require_grid_model(model)
    lo, hi = model.value_range
    meta = VolumeMeta(dims=dims, dtype="f32", value_range=(lo, hi))
    if to_host:
        return ScalarField(meta=meta, data=_decode_to_host(model, dims, slab_z))
    data = torch.empty((dz, dy, dx), dtype=torch.float32, device=model.flat_params.device)
    step = dz if slab_z is None else int(slab_z)
    if step < 1:
        raise ConfigError("slab_z must be >= 1")
    for z0 in range(0, dz, step):
        nz = min(step, dz - z0)
        decode_brick(model, dims, z0, nz, data[z0:z0 + nz])
    return ScalarField(meta=meta, data=data)


_HOST_SLAB_BYTES = 64 << 20     # device/pinned slab size of the host-landing decode
_HOST_RING = 4                  # slabs in flight (decode -> D2H -> host copy)


def _decode_to_host(model: NeuralModel, dims, slab_z=None) -> np.ndarray:
    """Decode into a host numpy array: a ring of device slabs + pinned staging slabs;
    slab k's decode (main stream) overlaps slab k-1's D2H (copy stream) and slab k-2's
    host copy into the output array (split over worker threads, GIL released by numpy).
    Measured at 1024^3 (tools/decode_e2e.py): the D2H runs at ~54 GB/s, one thread's copy
    into a fresh array at ~4.4 GB/s, so the copy is split: 0.38 s (4 threads, one per slab)
    -> 0.33 s (16 threads) against 0.317 s for the device-only decode."""
    from concurrent.futures import ThreadPoolExecutor
    dx, dy, dz = dims
    plane = dx * dy
    slab_bytes = int(os.environ.get("NVOL_DECODE_SLAB_MB", "0")) << 20 or _HOST_SLAB_BYTES
    nzs = int(slab_z) if slab_z else max(1, min(dz, slab_bytes // max(4 * plane, 1)))
    if nzs < 1:
        raise ConfigError("slab_z must be >= 1")
    out = np.empty((dz, dy, dx), dtype=np.float32)
    dev = model.flat_params.device
    nring = min(_HOST_RING, -(-dz // nzs))
    dbuf = [torch.empty((nzs, dy, dx), dtype=torch.float32, device=dev) for _ in range(nring)]
    hbuf = [torch.empty((nzs, dy, dx), dtype=torch.float32).pin_memory() for _ in range(nring)]
    decoded = [torch.cuda.Event() for _ in range(nring)]
    landed = [torch.cuda.Event() for _ in range(nring)]
    main = torch.cuda.current_stream()
    copy = torch.cuda.Stream(device=dev)
    pending = [[] for _ in range(nring)]
    # each slab's pinned -> output copy is split over several host threads: one thread's memcpy
    # (and the first touch of the output pages) runs far below the D2H rate
    workers = max(1, int(os.environ.get("NVOL_DECODE_HOST_THREADS", str(min(16, os.cpu_count() or 1)))))
    parts = max(1, workers // nring)

    def host_copy(k, z0, nz, a, b):
        landed[k].synchronize()
        flat_out = out[z0:z0 + nz].reshape(-1)
        np.copyto(flat_out[a:b], hbuf[k][:nz].numpy().reshape(-1)[a:b])

    with ThreadPoolExecutor(max_workers=max(workers, nring)) as pool:
        for i, z0 in enumerate(range(0, dz, nzs)):
            k = i % nring
            nz = min(nzs, dz - z0)
            for f in pending[k]:
                f.result()                      # pinned slot k is free again (its D2H landed too)
            decode_brick(model, dims, z0, nz, dbuf[k][:nz])
            decoded[k].record(main)
            copy.wait_event(decoded[k])
            with torch.cuda.stream(copy):
                hbuf[k][:nz].copy_(dbuf[k][:nz], non_blocking=True)
            landed[k].record(copy)              # (slot k is reused only after pending[k]: D2H + copy done)
            n = nz * plane
            cuts = [n * j // parts for j in range(parts + 1)]
            pending[k] = [pool.submit(host_copy, k, z0, nz, cuts[j], cuts[j + 1]) for j in range(parts)]
        for fs in pending:
            for f in fs:
                f.result()
    return out


def compression_ratio(model: NeuralModel, meta: VolumeMeta) -> float:
    """(source bytes) / (parameter bytes at f32) (trainer.py:109-111)."""
    return (meta.voxel_count * meta.itemsize) / (model.n_params * 4.0)


def save_model(model: NeuralModel, path) -> None:
    """trainer.py:125-138: magic, version, sorted-key config JSON, f32 blob."""
    if model.dtype != np.float32:
        raise ConfigError("only float32 models serialize; rebuild with dtype=float32")
    cfg = model.config_json()
    cfg["dims"] = list(model.dims)
    cfg["value_range"] = [model.value_range[0], model.value_range[1]]
    cfg["n_params"] = model.n_params
    blob = model.blob().cpu().numpy().astype("<f4")
    payload = json.dumps(cfg, sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MODEL_MAGIC)
        fh.write(struct.pack("<II", MODEL_VERSION, len(payload)))
        fh.write(payload)
        fh.write(blob.tobytes())


def load_model(path) -> NeuralModel:
    """trainer.py:141-171 (fresh optimizer state, as the reference)."""
    raw = Path(path).read_bytes()
    if len(raw) < 12 or raw[:4] != MODEL_MAGIC:
        raise FormatError(f"{path}: bad magic; not a model file")
    version, jlen = struct.unpack("<II", raw[4:12])
    if version != MODEL_VERSION:
        raise FormatError(f"{path}: unsupported version {version} (expected {MODEL_VERSION})")
    if len(raw) < 12 + jlen:
        raise FormatError(f"{path}: truncated config (expected {jlen} bytes, found {len(raw) - 12})")
    try:
        cfg = json.loads(raw[12:12 + jlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise FormatError(f"{path}: config block is not valid JSON ({exc})") from exc
    model = build_model(cfg, dims=tuple(cfg.get("dims", (2, 2, 2))),
                        value_range=tuple(cfg.get("value_range", (0.0, 1.0))))
    blob = np.frombuffer(raw[12 + jlen:], dtype="<f4")
    expected = model.n_params
    if "n_params" in cfg and cfg["n_params"] != expected:
        raise FormatError(f"{path}: header n_params {cfg['n_params']} != config-derived {expected}")
    if blob.size != expected:
        raise FormatError(f"{path}: parameter blob has {blob.size} floats, expected {expected}")
    model.load_blob(blob)
    return model
